import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch
from paper_2410_06106_b200 import configs as C, tomoq
cfg = C.C4(1)
inp = C.make_inputs(cfg, with_truth=False)
for ll in (0, 10, 20):
    ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule)
    ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
    ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=ll)
    ctx.set_sinogram(0, inp.sino[0])
    st = torch.cuda.Stream()
    ctx.run(5, st)
    ctx.launch_component(3, 5, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.launch_component(3, 20, st)
    e1.record(st)
    torch.cuda.synchronize()
    print("lloyd", ll, "encode us", round(e0.elapsed_time(e1) / 20 * 1e3, 1))
    ctx.close()

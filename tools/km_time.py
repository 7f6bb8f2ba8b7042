"""Time the K-means encode component (tq_launch_component 3) of the C4_G1 context alone."""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch
from paper_2410_06106_b200 import configs as C, tomoq
cfg = C.C4(1)
inp = C.make_inputs(cfg, with_truth=False)
ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule)
ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=cfg.lloyd)
ctx.set_sinogram(0, inp.sino[0])
st = torch.cuda.Stream()
ctx.run(5, st)
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.launch_component(3, 50, st)
    e1.record(st)
    torch.cuda.synchronize()
    print("kmeans encode us", round(e0.elapsed_time(e1) / 50 * 1e3, 1))

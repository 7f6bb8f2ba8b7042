"""Which public-API call of the bench's end-to-end loop costs device time (GPU box):
the asynchronous loop of bench.py with each part switched on in turn, CUDA events over 50 steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_06106_b200 import configs as C, tomoq  # noqa: E402

cfg = C.C4(1)
inp = C.make_inputs(cfg, with_truth=False)
ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule)
ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=cfg.lloyd)
sino = torch.from_numpy(inp.sino[0]).pin_memory()
img = [torch.empty(cfg.N * cfg.N, dtype=torch.float32).pin_memory() for _ in range(2)]
ctx.set_sinogram(0, sino)
st, cs = torch.cuda.Stream(), torch.cuda.Stream()
ctx.run(8, st)
torch.cuda.synchronize()
K = 48
for name, ss, im in (("run_async only", False, False), ("+ set_sinogram", True, False),
                     ("+ image_async", False, True), ("bench loop", True, True), ("run(48)", None, None)):
    for rep in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        if ss is None:
            ctx.run(K, st)
        else:
            for k in range(K):
                if ss:
                    ctx.set_sinogram(0, sino)
                ctx.run_async(1, st)
                if im:
                    ctx.image_async(img[k & 1], cs, 0, 0)
            ctx.wait()
        b.record(st)
        cs.synchronize()
        torch.cuda.synchronize()
    print(f"{name:16s} {a.elapsed_time(b) / K:.4f} ms per step")

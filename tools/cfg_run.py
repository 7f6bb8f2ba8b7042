"""A few ADMM iterations of one BASELINE config (for ncu launch lists on the GPU box).
PYTHONPATH=. python tools/cfg_run.py C2|C3|C5 [iters]"""
import sys

import torch

from paper_2410_06106_b200 import configs as C
from paper_2410_06106_b200 import tomoq

name = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = {"C1": C.C1, "C2": C.C2, "C3": C.C3, "C5": lambda: C.C5(slices=2)}[name]()
inp = C.make_inputs(cfg, with_truth=False)
ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule,
                    n_slices=len(inp.sino))
ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=cfg.lloyd, quality=cfg.quality)
for s, d in enumerate(inp.sino):
    ctx.set_sinogram(s, d)
ctx.run(iters)
torch.cuda.synchronize()
print(name, "ms/iter", ctx.stats()["ms_last_run"] / iters)

"""Config 3 with JPEG entropy-coded DCT payloads (restart 4): a few ADMM iterations, for
ncu launch lists (GPU box).  PYTHONPATH=. python tools/c3_jpeg_run.py [restart]"""
import sys

import torch

from paper_2410_06106_b200 import configs as C
from paper_2410_06106_b200 import tomoq

R = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = C.C3()
inp = C.make_inputs(cfg, with_truth=False)
ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule)
ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
ctx.set_quantizer(cfg.quant, quality=cfg.quality, jpeg_restart=R)
ctx.set_sinogram(0, torch.tensor(inp.sino[0], device="cuda"))
ctx.run(3)
torch.cuda.synchronize()
print("ms/iter", ctx.stats()["ms_last_run"] / 3)

"""Two profiled C4_G1 iterations (per-phase graphs, tq_set_profiling) for an ncu launch
list grouped by the engine's NVTX phase ranges:
ncu --nvtx --metrics gpu__time_duration.sum --csv python tools/nvtx_phases.py"""
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
ctx.set_sinogram(0, inp.sino[0])
ctx.run(2)
ctx.set_profiling(True)
ctx.run(2)
print({k: v for k, v in ctx.stats().items() if k.startswith("phase")})
ctx.close()

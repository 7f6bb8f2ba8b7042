"""DCT-J entropy coding on config 3 (GPU box): encode-stage time and bytes per restart
interval, and the whole ADMM iteration with and without entropy coding.
PYTHONPATH=. python tools/jpeg_probe.py"""
import torch

import bench
from paper_2410_06106_b200 import configs as C
from paper_2410_06106_b200 import tomoq

s = torch.cuda.Stream()
for R in (1, 2, 4, 8, 16):
    d = bench.dct_entropy_c3(tomoq, torch, s, restart=R)
    print(R, round(d["entropy"]["encode_us"], 1), d["entropy"]["payload_bytes_per_iter"],
          round(d["compression_vs_plain"], 2), "plain", round(d["plain"]["encode_us"], 1))
cfg = C.C3()
inp = C.make_inputs(cfg, with_truth=False)
for R in (0, 1, 4, 8):
    ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule)
    ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
    ctx.set_quantizer(cfg.quant, quality=cfg.quality, jpeg_restart=R)
    ctx.set_sinogram(0, torch.tensor(inp.sino[0], device="cuda"))
    ctx.run(3)
    ctx.run(10)
    print("C3 ADMM iteration, restart", R, round(ctx.stats()["ms_last_run"] / 10, 3), "ms")
    ctx.close()

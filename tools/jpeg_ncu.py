"""Config 3's DCT-J encode stage (restart 4) a few times, for an ncu launch list.
PYTHONPATH=. ncu --metrics gpu__time_duration.sum --csv python tools/jpeg_ncu.py"""
import torch

from paper_2410_06106_b200 import configs as C
from paper_2410_06106_b200 import tomoq

cfg = C.C3()
inp = C.make_inputs(cfg, with_truth=False)
ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule)
ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
ctx.set_quantizer(cfg.quant, quality=cfg.quality, jpeg_restart=4)
ctx.set_sinogram(0, torch.tensor(inp.sino[0], device="cuda"))
ctx.run(3)
s = torch.cuda.Stream()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("enc")
ctx.launch_component(4, 3, s)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
ctx.close()

"""Launch list of the forward projector component on C5's slice geometry (run under ncu
--metrics gpu__time_duration.sum): tile pass vs band reduction at 188 angles per node."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_06106_b200 import configs as C, synth, tomoq
cfg = C.C5(slices=1)
ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, synth.complete(cfg.nodes), split=cfg.split, rule=cfg.rule)
ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
ctx.set_quantizer(tomoq.Q_NONE)
ctx.set_sinogram(0, torch.rand(cfg.n_angles, cfg.n_det, device="cuda"))
s = torch.cuda.Stream()
ctx.launch_component(0, 3, s)
torch.cuda.synchronize()
ctx.close()

"""How much of a C4_G1 iteration (default node groups) each optional piece costs: the iteration
time with Lloyd steps 10 / 0, with K-means / no quantizer (CUDA events, 48 iterations)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_06106_b200 import configs as C, tomoq

cfg = C.C4(1)
inp = C.make_inputs(cfg, with_truth=False)

def t(quant, lloyd):
    ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule)
    ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
    ctx.set_quantizer(quant, k=cfg.k, lloyd=lloyd)
    ctx.set_sinogram(0, inp.sino[0])
    s = torch.cuda.Stream()
    ctx.run(8, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); ctx.run(48, s); b.record(s)
    torch.cuda.synchronize()
    g = ctx.stats()["node_groups"]
    ctx.close()
    return a.elapsed_time(b) / 48, g

for rep in range(2):
    for q, l in ((tomoq.Q_KMEANS, 10), (tomoq.Q_KMEANS, 0), (tomoq.Q_NONE, 10)):
        ms, g = t(q, l)
        print(f"quant {q} lloyd {l}: {ms:.4f} ms/iter (groups {g})", flush=True)

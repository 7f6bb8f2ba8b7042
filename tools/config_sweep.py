"""Iterations/s of every BASELINE config on one GPU (informational; bench.py is the headline).

python tools/config_sweep.py [--c5-slices 4]
Prints one JSON line per config: ms per ADMM iteration (CUDA events over `iters` iterations
after 2 warm-up iterations), G voxel-updates/s, and the K-means / DCT share is implicit.
C5 runs a subset of its 32 slices (same per-slice work; the full config is 32 slices)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2410_06106_b200 import configs as C  # noqa: E402
from paper_2410_06106_b200 import tomoq  # noqa: E402


def run(cfg, iters, slices=None):
    inp = C.make_inputs(cfg, with_truth=False, slices=slices)
    ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split, rule=cfg.rule,
                        n_slices=len(inp.sino))
    ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)
    ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=cfg.lloyd, quality=cfg.quality)
    for s, d in enumerate(inp.sino):
        ctx.set_sinogram(s, d)
    st = torch.cuda.Stream()
    ctx.run(2, st)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    ctx.run(iters, st)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    vu = 2 * (cfg.e1 + 1) * cfg.N * cfg.N * cfg.n_angles * len(inp.sino)
    ctx.close()
    return {"config": cfg.name, "N": cfg.N, "nodes": cfg.nodes, "slices": len(inp.sino), "quant": cfg.quant,
            "ms_per_iter": round(ms, 4), "admm_iters_per_s": round(1e3 / ms, 2), "gvu_s": round(vu / ms / 1e6, 1)}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--c5-slices", type=int, default=4)
    args = ap.parse_args()
    for make, it in ((C.C1, 50), (C.C2, 50), (C.C3, 20), (lambda: C.C4(1), 20)):
        print(json.dumps(run(make(), it)), flush=True)
    print(json.dumps(run(C.C5(slices=32), 3, slices=range(args.c5_slices))), flush=True)

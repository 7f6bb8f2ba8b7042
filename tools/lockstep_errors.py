"""Observed lockstep errors (SURVEY 8(c) parity item 4): for each config the oracle advances
one iteration from the GPU's exported state (fp32 production mode); the relative L2 error
of every node's next pre-quantization iterate is recorded, with the K-means label agreement
and the DCT decode equality.  Writes profiles/r2_lockstep_errors.json (tests/test_gpu_admm.py
bounds are set from these values)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
from paper_2410_06106_b200 import configs as C  # noqa: E402
from tests.cases import export_all, gpu_context, oracle_case, rel  # noqa: E402


def lockstep(cfg, inp, steps, warm, threads=8):
    ctx = gpu_context(cfg, inp, keep_labels=True)
    ctx.run(warm)
    out = []
    for _ in range(steps):
        X, L, XH = export_all(ctx, cfg)
        o = oracle_case(cfg, inp, threads=threads)
        o.X, o.L, o.XH = X.copy(), L.copy(), XH.copy()
        o.run(1)
        ctx.run(1)
        Xg, _, _ = export_all(ctx, cfg)
        errs = [rel(Xg[m], o.X[m]) for m in range(cfg.nodes)]
        rec = {"max_rel": max(errs), "median_rel": float(np.median(errs))}
        if cfg.quant == C.Q_KMEANS:
            ag = []
            for m in range(cfg.nodes):
                lab = ctx.labels(0, m, cfg.N * cfg.N)
                _, lr = oracle.kmeans_encode(Xg[m].astype(np.float32), cfg.k, cfg.lloyd)
                ag.append(float(np.mean(lab == lr)))
            rec["min_label_agreement"] = min(ag)
        out.append(rec)
    ctx.close()
    return out


def main():
    res = {"nproc": os.cpu_count()}
    cases = [("C2", C.C2(), 3, 2), ("C3", C.C3(), 3, 2), ("C4_G1", C.C4(1), 2, 2)]
    for name, cfg, steps, warm in cases:
        t0 = time.time()
        inp = C.make_inputs(cfg, with_truth=False)
        res[name] = lockstep(cfg, inp, steps, warm)
        res[name + "_seconds"] = round(time.time() - t0, 1)
        print(name, res[name], flush=True)
    os.makedirs("profiles", exist_ok=True)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/r2_lockstep_errors.json", "w"), indent=1)


if __name__ == "__main__":
    main()

"""the paper's experimental designs on a paper-shaped
synthetic workload, run through the hot path (libtomoq via the tomoq binding).

Workload W2 (R-27): a three-level phantom (synth.three_level_phantom) at 512^2,
804 angles evenly spaced in [0, 180), 725 detector bins (the paper pads the image
to 724^2 and records 724 bins; 725 is the smallest odd count covering the 512^2
image's diagonal, which our geometry check requires), continuous-model sinogram plus
Gaussian noise with sigma = NSD x max(d).

Designs reproduced (the numbers themselves live only in the paper's figures):
* CTR (Alg. 1) = one node, no edges, GD with E1 = 10 steps per outer iteration,
  warm start -- i.e. plain gradient descent on the whole sinogram.  Step: DESIGN.md R-8,
  eta_i = 1 / (2 a_i N + c_i), which at the paper's scale and one node is 1.2e-6 -- the
  paper's heuristic 1e-6 -- and scales with the node's angle count elsewhere;
* dADMM at 2 nodes (odd / even angles) and 10 nodes (81 x 4 + 80 x 6 round-robin,
  P:319-320), no quantization (Fig. 4), with the paper's rule (eq:solve_u..lamda, Alg. 3,
  E2 = 10, eta2 = 0.2) and the graph rule (R-7, ring);
* elbow sweep (Fig. 5): dADMM-K for K = 2..6 and dADMM-J for several qualities, RMSE vs
  compression (32 / ceil(log2 K) for K-means, payload bytes for the DCT);
* noise ladder (Figs. 6-7): NSD in {0, 0.24, 0.77, 2.43} % for dADMM-K (K = 3) and dADMM-J;
* convergence traces (Fig. 8): ||x_k - x_{k-1}|| / ||x_k|| per outer iteration.

RMSE and PSNR follow P:298-302 (PSNR with I_max = the true image's maximum)."""
from __future__ import annotations

import math
import time

import numpy as np

from . import configs as C
from . import synth, tomoq

NSD_LADDER = (0.0, 0.0024, 0.0077, 0.0243)


def paper_workload(N=512, n_angles=804, n_det=725, nsd=0.0, seed=7001):
    """(truth image, sinogram fp32 [n_angles][n_det]) of workload W2."""
    e = synth.three_level_phantom(N, seed)
    th = synth.default_angles(n_angles)
    d = synth.ellipse_sinogram(e, th, n_det)
    d = synth.add_noise(d, nsd, seed + 1)
    return synth.rasterize(e, N), d.astype(np.float32)


def rmse(x, truth):
    return float(np.sqrt(np.mean((np.asarray(x, np.float64) - truth) ** 2)))


def psnr(x, truth):
    r = rmse(x, truth)
    return float(20.0 * math.log10(float(truth.max()) / r)) if r > 0 else float("inf")


def run_case(truth, sino, n_angles, n_det, nodes, *, rule=C.RULE_GRAPH, inner=C.INNER_GD, e1=10,
             eta1=None, rho=1.0, e2=10, eta2=0.2, quant=C.Q_NONE, k=3, quality=50, iters=20,
             graph="ring", precision=0, trace=True, jpeg_restart=0):
    """One reconstruction through the C-ABI; returns the final image, RMSE/PSNR and the
    per-iteration convergence trace (||x_k - x_{k-1}|| / ||x_k||) and RMSE trace."""
    N = truth.shape[0]
    M = nodes
    edges = [] if M == 1 else (synth.make_graph(graph, M, 7003) if rule == C.RULE_GRAPH else synth.ring(M))
    ctx = tomoq.Context(N, n_angles, n_det, M, edges, split=C.SPLIT_RR, rule=rule, precision=precision)
    ctx.set_params(rho, inner=inner, e1=e1, eta1=[eta1] * M if (inner == C.INNER_GD and eta1) else None,
                   e2=e2, eta2=eta2)
    ctx.set_quantizer(quant, k=k, lloyd=10, quality=quality, jpeg_restart=jpeg_restart)
    ctx.set_sinogram(0, sino)
    prev = np.zeros(N * N)
    rel, err = [], []
    t0 = time.perf_counter()
    dev_ms = 0.0
    diverged = False
    try:
        for it in range(iters if trace else 1):
            ctx.run(1 if trace else iters)
            dev_ms += ctx.stats()["ms_last_run"]
            if trace:
                x = ctx.image().astype(np.float64).ravel()
                nx = np.linalg.norm(x)
                rel.append(float(np.linalg.norm(x - prev) / nx) if nx > 0 else 0.0)
                err.append(rmse(x.reshape(N, N), truth))
                prev = x
    except tomoq.TomoQError as exc:  # the paper rule can diverge
        if exc.code != 5:
            raise
        diverged = True
    x = ctx.image().reshape(N, N)
    st = ctx.stats()
    ctx.close()
    sends = 0 if M == 1 else (2 * len(edges) if rule == C.RULE_GRAPH else M * (M - 1))
    return {"nodes": M, "rule": rule, "quant": quant, "k": k, "quality": quality, "iters": iters,
            "diverged": diverged, "rmse": rmse(x, truth), "psnr": psnr(x, truth), "rel_change": rel,
            "rmse_trace": err, "payload_bytes_per_iter": int(st["payload_bytes_logical"]),
            "compression_percent": compression_percent(int(st["payload_bytes_logical"]), sends, N * N)
            if sends else None,
            "device_ms": dev_ms, "wall_s": time.perf_counter() - t0, "image": x}


def compression_percent(payload_bytes_per_iter, sends_per_iter, n):
    """1 - (bytes of one payload) / (4 n bytes of the fp32 vector), in percent.  (P:345
    quotes 90.6% for K = 3 and 85.3% for K = 32 at "2-bit and 5-bit precision"; those two
    figures do not follow one formula, so the measured payload size is reported.)"""
    return 100.0 * (1.0 - payload_bytes_per_iter / max(1, sends_per_iter) / (4.0 * n))


def studies(scale="reduced", iters=None, seed=7001):
    """All four designs; scale 'full' = 512^2 / 804 angles, 'reduced' = 128^2 / 201 angles
    (same structure, minutes instead of hours).  Returns a JSON-able dict."""
    if scale == "full":
        N, n_ang, n_det = 512, 804, 725
        it = iters or 1000  # 1000 outer iterations for the Phantom
    else:
        N, n_ang, n_det = 128, 201, 183
        it = iters or 300
    out = {"workload": {"N": N, "n_angles": n_ang, "n_det": n_det, "phantom": "three-level (synth)",
                        "inner": "GD E1=10, eta1 = 1/(2 a_i N + c_i) (R-8)", "outer_iters": it}}
    truth, sino = paper_workload(N, n_ang, n_det, 0.0, seed)
    strip = lambda r: {k: v for k, v in r.items() if k != "image"}  # noqa: E731
    # Fig. 4: CTR vs dADMM at 2 and 10 nodes, unquantized
    fig4 = {"ctr": strip(run_case(truth, sino, n_ang, n_det, 1, iters=it))}
    for M in (2, 10):
        for rule, name in ((C.RULE_PAPER, "paper_rule"), (C.RULE_GRAPH, "graph_rule")):
            fig4[f"dadmm_{M}_{name}"] = strip(run_case(truth, sino, n_ang, n_det, M, rule=rule, iters=it))
    out["fig4_ctr_vs_dadmm"] = fig4
    # Fig. 5: elbow sweep (10 nodes, graph rule)
    fig5 = {"kmeans": [], "dct": []}
    for K in range(2, 7):
        r = run_case(truth, sino, n_ang, n_det, 10, quant=C.Q_KMEANS, k=K, iters=it)
        fig5["kmeans"].append({"K": K, "compression_percent": r["compression_percent"], "rmse": r["rmse"],
                               "psnr": r["psnr"]})
    for q in (5, 10, 25, 50, 75, 90):  # DCT payloads entropy-coded (NEXT-2) so the bytes are real
        r = run_case(truth, sino, n_ang, n_det, 10, quant=C.Q_DCT, quality=q, iters=it, jpeg_restart=4)
        fig5["dct"].append({"quality": q, "compression_percent": r["compression_percent"], "rmse": r["rmse"],
                            "psnr": r["psnr"]})
    out["fig5_elbow"] = fig5
    # Figs. 6-8: noise ladder with K = 3 and DCT quality 50, convergence traces
    fig6 = []
    for nsd in NSD_LADDER:
        t2, s2 = paper_workload(N, n_ang, n_det, nsd, seed)
        for quant, name in ((C.Q_KMEANS, "dADMM-K"), (C.Q_DCT, "dADMM-J")):
            r = run_case(t2, s2, n_ang, n_det, 10, quant=quant, k=3, quality=50, iters=it, jpeg_restart=4)
            fig6.append({"nsd_percent": 100 * nsd, "method": name, "rmse": r["rmse"], "psnr": r["psnr"],
                         "rel_change": r["rel_change"], "rmse_trace": r["rmse_trace"]})
    out["fig6_8_noise_and_convergence"] = fig6
    return out

"""Builds the same ADMM case on the CUDA path (through the C-ABI) and on the oracle,
from one set of seeded synthetic inputs (paper_2410_06106_b200.synth)."""
import numpy as np

import oracle
from paper_2410_06106_b200 import configs as C
from paper_2410_06106_b200 import tomoq

QKIND = {C.Q_NONE: 0, C.Q_KMEANS: 1, C.Q_DCT: 2}


def slice_kind(cfg, s):
    if cfg.quant == C.Q_ALT:
        return C.Q_KMEANS if s % 2 == 0 else C.Q_DCT
    return cfg.quant


def gpu_context(cfg, inp, precision=0, keep_labels=False, eta1=None, angles=None, stop_tol=0.0):
    ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split,
                        rule=cfg.rule, n_slices=len(inp.sino), precision=precision, projector=cfg.projector,
                        angles=angles)
    ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1, eta1=eta1, e2=cfg.e2, eta2=cfg.eta2, stop_tol=stop_tol)
    ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=cfg.lloyd, quality=cfg.quality, keep_labels=keep_labels,
                      jpeg_restart=cfg.jpeg_restart)
    for s, d in enumerate(inp.sino):
        ctx.set_sinogram(s, d)
    return ctx


def oracle_case(cfg, inp, s=0, threads=8, eta1=None, theta=None, stop_tol=0.0):
    return oracle.OracleADMM(cfg.N, cfg.n_det, cfg.n_angles, cfg.nodes, inp.edges,
                             inp.sino[s].astype(np.float64), cfg.split == C.SPLIT_CONTIG,
                             rule=cfg.rule, inner=cfg.inner, e1=cfg.e1, rho=cfg.rho, eta1=eta1,
                             e2=cfg.e2, eta2=cfg.eta2, qkind=QKIND[slice_kind(cfg, s)], K=cfg.k,
                             lloyd=cfg.lloyd, quality=cfg.quality, threads=threads, projector=cfg.projector,
                             theta=theta, stop_tol=stop_tol)


def export_all(ctx, cfg, s=0):
    """GPU state of every node of slice s as the oracle's (X, L, XH) arrays."""
    n = cfg.N * cfg.N
    X = np.zeros((cfg.nodes, n)); L = np.zeros((cfg.nodes, n))
    XH = np.zeros((cfg.nodes if cfg.rule == C.RULE_GRAPH else 1, n))
    for m in range(cfg.nodes):
        st = ctx.export_state(s, m)
        X[m], L[m] = st[0], st[1]
        if cfg.rule == C.RULE_GRAPH:
            XH[m] = st[2]
        else:
            XH[0] = st[2]
    return X, L, XH


def rel(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))

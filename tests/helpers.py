"""Test-only helpers that do not depend on oracle.c or the CUDA path."""
import math

import numpy as np


def dense_joseph(N, n_ang, n_det, sel=None):
    """Brute-force Joseph system matrix from the geometry: walk each ray's
    major-axis pixel lines and give each pixel its linear-interpolation weight
    times the per-line ray length 1/m (rows: selected angles x bins)."""
    sel = list(range(n_ang)) if sel is None else list(sel)
    A = np.zeros((len(sel) * n_det, N * N))
    half = (N - 1) / 2.0
    for k, a in enumerate(sel):
        th = math.pi * a / n_ang
        c, s = math.cos(th), math.sin(th)
        xmaj = 4 * a >= n_ang and 4 * a <= 3 * n_ang
        cols = np.arange(N)
        for j in range(n_det):
            t = j - (n_det - 1) / 2.0
            row = A[k * n_det + j].reshape(N, N)
            if not xmaj:
                for r in range(N):
                    col = (t - (half - r) * s) / c + half
                    row[r, :] += np.maximum(0.0, 1.0 - np.abs(col - cols)) / abs(c)
            else:
                for cc in range(N):
                    rr = half - (t - (cc - half) * c) / s
                    row[:, cc] += np.maximum(0.0, 1.0 - np.abs(rr - cols)) / abs(s)
    return A


def rel(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)

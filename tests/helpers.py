"""Test-only helpers that do not depend on oracle.c or the CUDA path."""
import math

import numpy as np


def dense_joseph(N, n_ang, n_det, sel=None, theta=None):
    """Brute-force Joseph system matrix from the geometry: walk each ray's
    major-axis pixel lines and give each pixel its linear-interpolation weight
    times the per-line ray length 1/m (rows: selected angles x bins).  theta: an
    explicit angle list (radians; major axis x iff |sin| >= |cos|, R-3)."""
    sel = list(range(n_ang)) if sel is None else list(sel)
    A = np.zeros((len(sel) * n_det, N * N))
    half = (N - 1) / 2.0
    for k, a in enumerate(sel):
        th = math.pi * a / n_ang if theta is None else float(theta[a])
        c, s = math.cos(th), math.sin(th)
        xmaj = (4 * a >= n_ang and 4 * a <= 3 * n_ang) if theta is None else abs(s) >= abs(c)
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


def clip_length(px0, px1, py0, py1, x0, y0, dx, dy):
    """Length of the line {(x0, y0) + a (dx, dy)} (unit direction) inside the closed box
    [px0, px1] x [py0, py1] (Liang-Barsky clipping of the infinite line)."""
    lo, hi = -math.inf, math.inf
    for p0, p1, o, d in ((px0, px1, x0, dx), (py0, py1, y0, dy)):
        if d == 0.0:
            if o < p0 or o > p1:
                return 0.0
            continue
        a1, a2 = (p0 - o) / d, (p1 - o) / d
        lo, hi = max(lo, min(a1, a2)), min(hi, max(a1, a2))
    return max(0.0, hi - lo)


def dense_siddon(N, n_ang, n_det, theta=None):
    """Exact intersection-length matrix by clipping every ray against every pixel square
    (no Siddon crossing lists); a ray lying on the edge shared by two pixels is counted
    half in each (R-26), trig exact at 0 and pi/2 (explicit lists: theta == 0,
    theta == fl64(pi/2))."""
    h = N / 2.0
    A = np.zeros((n_ang * n_det, N * N))
    for a in range(n_ang):
        th = math.pi * a / n_ang if theta is None else float(theta[a])
        zero = a == 0 if theta is None else th == 0.0
        half_pi = 2 * a == n_ang if theta is None else th == math.pi / 2
        if zero:
            cs, sn = 1.0, 0.0
        elif half_pi:
            cs, sn = 0.0, 1.0
        else:
            cs, sn = math.cos(th), math.sin(th)
        for j in range(n_det):
            t = j - 0.5 * (n_det - 1)
            x0, y0, dx, dy = t * cs, t * sn, -sn, cs
            for r in range(N):
                for c in range(N):
                    bx0, bx1 = c - h, c + 1 - h
                    by0, by1 = h - r - 1, h - r
                    ln = clip_length(bx0, bx1, by0, by1, x0, y0, dx, dy)
                    if ln > 0 and ((dx == 0 and x0 in (bx0, bx1)) or (dy == 0 and y0 in (by0, by1))):
                        ln *= 0.5  # on an edge: the closed squares on both sides both contain it
                    A[a * n_det + j, r * N + c] = ln
    return A

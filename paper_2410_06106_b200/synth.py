"""Seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This module holds NONE of the method's arithmetic (no Joseph projector, no ADMM,
no quantizer).  It only draws the stand-in data the paper's experiments need
("Phantom image ... 32-bits precision", PAPER.md:349-353 Gaussian
sinogram noise) and the communication graphs BASELINE.json's configs name:

* ellipse phantoms (centres/axes/angles/intensities drawn from numpy PCG64),
* their *continuous* x-ray transform (Eq. 1) evaluated in closed form
  (chord length of an ellipse) -- i.e. the data come from the continuous model,
  not from the discrete system matrix the method uses (no "inverse crime"),
* an optional pixel-square texture (config 3) whose continuous transform is the
  exact trapezoid footprint of each square pixel,
* i.i.d. Gaussian noise with sigma = p * max(d_clean) (PAPER.md:351 NSD, R-14),
* graphs: ring, 2-D torus, random d-regular (configuration model), complete.

The recipe (ranges, seeds) is stated in DESIGN.md "Input recipe".
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


# ----------------------------------------------------------------------------- phantoms
@dataclass
class Ellipses:
    x0: np.ndarray
    y0: np.ndarray
    a: np.ndarray
    b: np.ndarray
    phi: np.ndarray
    rho: np.ndarray

    def __len__(self):
        return len(self.x0)


def random_ellipses(n_ellipses: int, N: int, seed: int) -> Ellipses:
    """Semi-axes a, b ~ U[0.05R, 0.5R] (R = N/2); centre uniform in the disk of
    radius 0.9R - max(a, b) so every ellipse lies inside the inscribed circle;
    rotation phi ~ U[0, pi); intensity ~ U[0.1, 1] (BASELINE.json configs)."""
    g = _rng(seed)
    R = N / 2.0
    a = g.uniform(0.05 * R, 0.5 * R, n_ellipses)
    b = g.uniform(0.05 * R, 0.5 * R, n_ellipses)
    rad = np.sqrt(g.uniform(0.0, 1.0, n_ellipses)) * (0.9 * R - np.maximum(a, b))
    ang = g.uniform(0.0, 2.0 * np.pi, n_ellipses)
    phi = g.uniform(0.0, np.pi, n_ellipses)
    rho = g.uniform(0.1, 1.0, n_ellipses)
    return Ellipses(rad * np.cos(ang), rad * np.sin(ang), a, b, phi, rho)


def three_level_phantom(N: int, seed: int) -> Ellipses:
    """Paper-shaped stand-in for the ToMoBAR Phantom ("three
    distinct gray levels"): a body ellipse of level 0.5 (semi-axes 0.80R x 0.68R, tilted
    0.1 rad) holding 5..8 disjoint inner ellipses that add 0.5 (level 1.0) -- background 0,
    body 0.5, features 1.0.  Inner semi-axes ~ U[0.06R, 0.22R], centres drawn until the
    inner ellipses' bounding circles are disjoint and inside 0.85 of the body."""
    g = _rng(seed)
    R = N / 2.0
    x0, y0, a, b, phi, rho = [0.0], [0.0], [0.80 * R], [0.68 * R], [0.1], [0.5]
    n_in = int(g.integers(5, 9))
    circles = []
    tries = 0
    while len(circles) < n_in and tries < 10000:
        tries += 1
        ai, bi = g.uniform(0.06 * R, 0.22 * R), g.uniform(0.06 * R, 0.22 * R)
        r = max(ai, bi)
        ang, rad = g.uniform(0, 2 * np.pi), np.sqrt(g.uniform()) * 0.85 * (0.68 * R - r)
        cx, cy = rad * np.cos(ang), rad * np.sin(ang)
        if all(math.hypot(cx - x, cy - y) > r + q + 1.0 for x, y, q in circles):
            circles.append((cx, cy, r))
            x0.append(cx); y0.append(cy); a.append(ai); b.append(bi)
            phi.append(g.uniform(0, np.pi)); rho.append(0.5)
    return Ellipses(np.array(x0), np.array(y0), np.array(a), np.array(b), np.array(phi), np.array(rho))


def pixel_centres(N: int):
    """x_c = c - (N-1)/2 (c = column), y_r = (N-1)/2 - r (r = row, row 0 on top)."""
    c = np.arange(N, dtype=np.float64)
    return c - (N - 1) / 2.0, (N - 1) / 2.0 - c


def rasterize(e: Ellipses, N: int, supersample: int = 4) -> np.ndarray:
    """Ground-truth image: ellipse intensities add; each pixel is the mean over a
    supersample x supersample grid of sub-pixel points.  Returns float64 N x N."""
    xs, ys = pixel_centres(N)
    off = (np.arange(supersample) + 0.5) / supersample - 0.5
    img = np.zeros((N, N), np.float64)
    for k in range(len(e)):
        rmax = max(e.a[k], e.b[k]) + 1.0
        c_lo = max(0, int(math.floor(e.x0[k] - rmax + (N - 1) / 2.0)))
        c_hi = min(N, int(math.ceil(e.x0[k] + rmax + (N - 1) / 2.0)) + 1)
        r_lo = max(0, int(math.floor((N - 1) / 2.0 - e.y0[k] - rmax)))
        r_hi = min(N, int(math.ceil((N - 1) / 2.0 - e.y0[k] + rmax)) + 1)
        X = xs[c_lo:c_hi][None, :, None, None] + off[None, None, None, :]
        Y = ys[r_lo:r_hi][:, None, None, None] - off[None, None, :, None]
        dx, dy = X - e.x0[k], Y - e.y0[k]
        cp, sp = math.cos(e.phi[k]), math.sin(e.phi[k])
        u = (dx * cp + dy * sp) / e.a[k]
        v = (-dx * sp + dy * cp) / e.b[k]
        inside = (u * u + v * v) <= 1.0
        img[r_lo:r_hi, c_lo:c_hi] += e.rho[k] * inside.mean(axis=(2, 3))
    return img


def texture(N: int, sigma: float, seed: int) -> np.ndarray:
    """i.i.d. N(0, sigma^2) per pixel (config 3 'seeded Gaussian texture')."""
    return _rng(seed).normal(0.0, sigma, (N, N))


# ----------------------------------------------------------------------------- continuous transform
def default_angles(n_angles: int) -> np.ndarray:
    """theta_a = pi * a / n_angles, evenly spaced in [0, 180)."""
    return np.pi * np.arange(n_angles, dtype=np.float64) / n_angles


def bin_centres(n_det: int) -> np.ndarray:
    """t_j = j - (n_det-1)/2, unit spacing."""
    return np.arange(n_det, dtype=np.float64) - (n_det - 1) / 2.0


def ellipse_sinogram(e: Ellipses, thetas: np.ndarray, n_det: int) -> np.ndarray:
    """Closed-form line integrals of the ellipse sum along the rays of Eq. 1
    (PAPER.md:42): ray (theta, t) = {p : p . (cos theta, sin theta) = t}.
    For one ellipse: tau = t - x0 cos - y0 sin, s^2 = a^2 cos^2(theta-phi) +
    b^2 sin^2(theta-phi); integral = rho * 2ab sqrt(s^2 - tau^2) / s^2 for |tau| < s."""
    t = bin_centres(n_det)[None, :]
    out = np.zeros((len(thetas), n_det), np.float64)
    ct, st = np.cos(thetas)[:, None], np.sin(thetas)[:, None]
    for k in range(len(e)):
        tau = t - e.x0[k] * ct - e.y0[k] * st
        d = thetas[:, None] - e.phi[k]
        s2 = (e.a[k] * np.cos(d)) ** 2 + (e.b[k] * np.sin(d)) ** 2
        out += e.rho[k] * 2.0 * e.a[k] * e.b[k] * np.sqrt(np.maximum(s2 - tau * tau, 0.0)) / s2
    return out


def pixel_square_sinogram(img: np.ndarray, thetas: np.ndarray, n_det: int) -> np.ndarray:
    """Continuous x-ray transform of a piecewise-constant image made of unit
    squares, sampled at bin centres.  The chord-length profile of one unit square
    at angle theta is the density of U1 cos + U2 sin (U ~ U[-1/2, 1/2]): a
    trapezoid of area 1 with half-widths (wmax -/+ wmin)/2, wmax/wmin = the larger/
    smaller of |cos|, |sin|."""
    N = img.shape[0]
    xs, ys = pixel_centres(N)
    X, Y = np.meshgrid(xs, ys)  # Y varies along rows
    vals = img.ravel()
    t0 = -(n_det - 1) / 2.0
    out = np.zeros((len(thetas), n_det), np.float64)
    for ia, th in enumerate(thetas):
        c, s = math.cos(th), math.sin(th)
        wmax, wmin = max(abs(c), abs(s)), min(abs(c), abs(s))
        tp = (X * c + Y * s).ravel()
        half = 0.5 * (wmax + wmin)
        jlo = np.floor(tp - half - t0).astype(np.int64)
        for dj in range(0, 3):
            j = jlo + dj
            tau = np.abs(t0 + j - tp)
            if wmin < 1e-12:
                w = (tau < 0.5 * wmax).astype(np.float64) / wmax
            else:
                w = np.clip((half - tau) / wmin, 0.0, 1.0) / wmax
            ok = (j >= 0) & (j < n_det) & (w > 0)
            out[ia] += np.bincount(j[ok], weights=(w * vals)[ok], minlength=n_det)
    return out


def add_noise(d_clean: np.ndarray, frac: float, seed: int) -> np.ndarray:
    """d = d_clean + N(0, sigma^2), sigma = frac * max(d_clean) (PAPER.md:351,
    NSD = sigma / x_peak; the configs state sigma as a % of the maximum)."""
    if frac == 0.0:
        return d_clean.copy()
    sigma = frac * float(np.max(d_clean))
    return d_clean + _rng(seed).normal(0.0, sigma, d_clean.shape)


# ----------------------------------------------------------------------------- graphs
def ring(M: int):
    if M <= 1:
        return []
    if M == 2:
        return [(0, 1)]
    return sorted({tuple(sorted((i, (i + 1) % M))) for i in range(M)})


def torus(rows: int, cols: int):
    """2-D torus, node id = cols * r + c, neighbours (r+-1, c), (r, c+-1) mod size."""
    E = set()
    for r in range(rows):
        for c in range(cols):
            i = cols * r + c
            for (rr, cc) in (((r + 1) % rows, c), (r, (c + 1) % cols)):
                j = cols * rr + cc
                if i != j:
                    E.add(tuple(sorted((i, j))))
    return sorted(E)


def complete(M: int):
    return [(i, j) for i in range(M) for j in range(i + 1, M)]


def _connected(M: int, edges) -> bool:
    adj = [[] for _ in range(M)]
    for i, j in edges:
        adj[i].append(j)
        adj[j].append(i)
    seen, stack = {0}, [0]
    while stack:
        u = stack.pop()
        for v in adj[u]:
            if v not in seen:
                seen.add(v)
                stack.append(v)
    return len(seen) == M


def random_regular(M: int, d: int, seed: int, max_tries: int = 100000):
    """Random simple connected d-regular graph by the configuration model with
    rejection (stubs shuffled by a seeded PCG64 stream, retried until simple and
    connected)."""
    assert (M * d) % 2 == 0 and d < M
    g = _rng(seed)
    stubs = np.repeat(np.arange(M), d)
    for _ in range(max_tries):
        perm = g.permutation(stubs)
        pairs = perm.reshape(-1, 2)
        if np.any(pairs[:, 0] == pairs[:, 1]):
            continue
        E = {tuple(sorted(map(int, p))) for p in pairs}
        if len(E) != len(pairs):
            continue
        E = sorted(E)
        if _connected(M, E):
            return E
    raise RuntimeError("no simple connected regular graph found")


def make_graph(kind: str, M: int, seed: int = 0):
    if kind == "ring":
        return ring(M)
    if kind == "torus":
        r = int(round(math.sqrt(M)))
        assert r * r == M, "torus needs a square node count"
        return torus(r, r)
    if kind == "regular4":
        return random_regular(M, 4, seed)
    if kind == "complete":
        return complete(M)
    if kind == "none":
        return []
    raise ValueError(kind)

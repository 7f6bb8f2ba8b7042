"""The five workloads of BASELINE.json "configs" (C1..C5), with every value the
config leaves unstated filled in per DESIGN.md "Readings".

A config is plain data; `make_inputs` draws its seeded synthetic inputs through
`synth` (phantom, continuous-model sinogram, noise, graph)."""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import synth

RULE_GRAPH, RULE_PAPER, RULE_CONSENSUS = 0, 1, 2
INNER_GD, INNER_CG = 0, 1
SPLIT_RR, SPLIT_CONTIG = 0, 1
Q_NONE, Q_KMEANS, Q_DCT, Q_ALT = 0, 1, 2, 3


@dataclass
class Config:
    name: str
    N: int
    n_ellipses: int
    n_angles: int
    n_det: int
    noise: float
    nodes: int
    graph: str
    split: int
    rho: float
    iters: int
    inner: int = INNER_CG
    e1: int = 5
    quant: int = Q_NONE
    k: int = 16
    lloyd: int = 10
    quality: int = 50
    projector: int = 0     # 0 Joseph (R-1), 1 Siddon (R-26, NEXT-3)
    jpeg_restart: int = 0  # DCT payloads: 0 plain int16 coefficients, R > 0 JPEG entropy coding (NEXT-2)
    texture: float = 0.0
    slices: int = 1
    rule: int = RULE_GRAPH
    e2: int = 10
    eta2: float = 0.2
    cid: int = 0
    extra: dict = field(default_factory=dict)

    def seeds(self, s: int = 0):
        """phantom, noise, graph, texture seeds (DESIGN.md input recipe)."""
        if self.slices > 1:
            return (5001 + 100 * s, 5002 + 100 * s, 1000 * self.cid + 3, 5004 + 100 * s)
        c = self.cid
        return (1000 * c + 1, 1000 * c + 2, 1000 * c + 3, 1000 * c + 4)


def n_det_for(N: int) -> int:
    """Smallest odd n_det >= ceil(N*sqrt(2)) (all configs already satisfy it)."""
    n = int(math.ceil(N * math.sqrt(2.0)))
    return n if n % 2 == 1 else n + 1


def C1():
    return Config("C1", N=64, n_ellipses=5, n_angles=90, n_det=91, noise=0.01, nodes=4,
                  graph="ring", split=SPLIT_CONTIG, rho=1.0, iters=20, cid=1)


def C2():
    return Config("C2", N=256, n_ellipses=20, n_angles=180, n_det=363, noise=0.01, nodes=8,
                  graph="ring", split=SPLIT_RR, rho=1.0, iters=50, quant=Q_KMEANS, k=16,
                  lloyd=10, cid=2)


def C3():
    return Config("C3", N=512, n_ellipses=40, n_angles=360, n_det=725, noise=0.01, nodes=16,
                  graph="torus", split=SPLIT_RR, rho=1.0, iters=100, quant=Q_DCT, quality=50,
                  texture=0.02, cid=3)


def C4(G: int = 8):
    """Weak-scaling config: M = 8G nodes, 90G angles (12/11 per node), 8 nodes/GPU."""
    return Config(f"C4_G{G}", N=1024, n_ellipses=60, n_angles=90 * G, n_det=1449, noise=0.005,
                  nodes=8 * G, graph="regular4", split=SPLIT_RR, rho=1.0, iters=100,
                  quant=Q_KMEANS, k=64, lloyd=10, cid=4, extra={"G": G})


def C5(slices: int = 32):
    """32 independent 2048^2 slices, 8 nodes/slice on a complete graph; even
    slices K-means K=32, odd slices DCT q75 (reading C-20)."""
    return Config("C5", N=2048, n_ellipses=60, n_angles=1500, n_det=2897, noise=0.01, nodes=8,
                  graph="complete", split=SPLIT_RR, rho=1.0, iters=50, quant=Q_ALT, k=32,
                  lloyd=10, quality=75, slices=slices, cid=5)


CONFIGS = {"C1": C1, "C2": C2, "C3": C3, "C4": C4, "C5": C5}


def scaled(cfg: Config, N: int, n_angles: int | None = None, **kw) -> Config:
    """Same structure at a smaller image (for oracle-speed parity cases)."""
    na = n_angles if n_angles is not None else cfg.n_angles
    return replace(cfg, N=N, n_angles=na, n_det=n_det_for(N), **kw)


@dataclass
class Inputs:
    cfg: Config
    truth: list          # per slice float64 N x N
    sino: list           # per slice float32 [n_angles][n_det] (noisy)
    edges: list          # undirected (i, j) pairs


def make_inputs(cfg: Config, with_truth: bool = True, slices=None) -> Inputs:
    sl = range(cfg.slices) if slices is None else slices
    truth, sino = [], []
    thetas = synth.default_angles(cfg.n_angles)
    for s in sl:
        ps, ns, _, ts = cfg.seeds(s)
        e = synth.random_ellipses(cfg.n_ellipses, cfg.N, ps)
        d = synth.ellipse_sinogram(e, thetas, cfg.n_det)
        img = synth.rasterize(e, cfg.N) if (with_truth or cfg.texture > 0) else None
        if cfg.texture > 0:
            tex = synth.texture(cfg.N, cfg.texture, ts)
            img = img + tex
            d = d + synth.pixel_square_sinogram(tex, thetas, cfg.n_det)
        d = synth.add_noise(d, cfg.noise, ns)
        truth.append(img)
        sino.append(d.astype(np.float32))
    edges = synth.make_graph(cfg.graph, cfg.nodes, cfg.seeds()[2])
    return Inputs(cfg, truth, sino, edges)

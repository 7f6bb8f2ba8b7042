"""The C-ABI fields beyond the first round's boundary: explicit angle lists
(tq_geometry.angles_rad), the relative-change stop (tq_params.stop_tol), the
per-node byte accounting of PAPER.md:248-252 (tq_get_node_bytes) and per-phase device time
(tq_set_profiling / tq_stats.phase_ms) -- each against the oracle or the paper's model."""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2410_06106_b200 import configs as C
from paper_2410_06106_b200 import synth
from paper_2410_06106_b200 import tomoq
from tests.cases import gpu_context, oracle_case, rel

pytestmark = pytest.mark.gpu


def irregular_angles(n, seed):
    """Seeded irregular angles in [0, pi) with the special ones (0, pi/4, pi/2, 3pi/4)."""
    rng = np.random.default_rng(seed)
    return np.concatenate([[0.0, math.pi / 4, math.pi / 2, 3 * math.pi / 4], rng.uniform(0, math.pi, n - 4)])


def jittered_angles(n, seed):
    """Seeded irregular but well spread angles: pi (a + U(-0.4, 0.4)) / n in [0, pi), with 0 and
    pi/2 exactly (the axis rays)."""
    rng = np.random.default_rng(seed)
    t = np.mod(math.pi * (np.arange(n) + rng.uniform(-0.4, 0.4, n)) / n, math.pi)
    t[0], t[n // 2] = 0.0, math.pi / 2
    return t


@pytest.mark.parametrize("N,n_ang,n_det", [(64, 40, 91), (200, 77, 285)])
@pytest.mark.parametrize("projector", [0, 1])
def test_explicit_angles_projector_parity(N, n_ang, n_det, projector):
    theta = irregular_angles(n_ang, N)
    rng = np.random.default_rng(N)
    x = rng.random((N, N))
    y = rng.random((n_ang, n_det))
    fo = oracle.project_siddon if projector else oracle.project
    bo = oracle.backproject_siddon if projector else oracle.backproject
    ref_f = fo(x, n_ang, n_det, theta=theta)
    ref_b = bo(y, N, n_ang, theta=theta)
    for dt, tol in ((torch.float32, 1e-5), (torch.float64, 1e-12)):
        f = tomoq.project(torch.tensor(x, dtype=dt, device="cuda"), n_ang, n_det, projector=projector, angles=theta)
        b = tomoq.backproject(torch.tensor(y, dtype=dt, device="cuda"), N, n_ang, projector=projector, angles=theta)
        assert rel(f.cpu().numpy(), ref_f) <= tol
        assert rel(b.cpu().numpy(), ref_b) <= tol


def explicit_c1(theta):
    cfg = C.C1()
    cfg.n_angles = len(theta)
    e = synth.random_ellipses(cfg.n_ellipses, cfg.N, 1001)
    d = synth.add_noise(synth.ellipse_sinogram(e, theta, cfg.n_det), cfg.noise, 1002)
    inp = C.Inputs(cfg, [synth.rasterize(e, cfg.N)], [d.astype(np.float32)], synth.make_graph("ring", 4, 1003))
    return cfg, inp


@pytest.mark.parametrize("prec,tol", [(0, 1e-3), (1, 1e-6)])
def test_explicit_angles_admm_c1(prec, tol):
    """Config 1 with 90 jittered angles (tq_geometry.angles_rad): the whole ADMM run against
    the oracle run with the same angle list."""
    theta = jittered_angles(90, 17)
    cfg, inp = explicit_c1(theta)
    ctx = gpu_context(cfg, inp, precision=prec, angles=theta)
    ctx.run(cfg.iters)
    o = oracle_case(cfg, inp, theta=theta).run(cfg.iters)
    assert rel(ctx.image(), o.image()) <= tol


@pytest.mark.parametrize("rule,tol", [(C.RULE_GRAPH, 2e-2), (C.RULE_CONSENSUS, 3e-3)])
def test_stop_tol_stops_where_the_oracle_does(rule, tol):
    """tq_params.stop_tol (R-13), fp64 verification mode: the GPU stops after the same
    iteration as the oracle, with the same iterates (1e-6) and relative change (a difference
    of nearly equal iterates: 1e-4)."""
    cfg = C.C1()
    cfg.rule = rule
    inp = C.make_inputs(cfg)
    ctx = gpu_context(cfg, inp, precision=1, stop_tol=tol)
    ctx.run(200)
    st = ctx.stats()
    o = oracle_case(cfg, inp, stop_tol=tol).run(200)
    assert 2 < o.last_run_iters < 200
    assert st["iters_last_run"] == o.last_run_iters
    assert abs(st["rel_change_last"] - o.last_change) <= 1e-4 * o.last_change
    X = np.stack([ctx.export_state(0, m)[0] for m in range(cfg.nodes)])  # fp64 state
    assert rel(X, o.X) <= 1e-6  # fp64 vs fp64 after ~50-70 iterations (CG amplifies rounding)
    # a second run continues from there (one more iteration already satisfies the test or not)
    ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1)  # stop_tol = 0: fixed count again
    ctx.run(3)
    assert ctx.stats()["iters_last_run"] == 3


def test_stop_tol_multirank_loopback():
    """The stop test is maximised over ranks (world 2, loopback): same stopping iteration and
    bitwise the same iterates as world 1."""
    from tests.test_gpu_multirank import node_images, run_world
    cfg = C.C2()
    inp = C.make_inputs(cfg, with_truth=False)
    tol = 2e-2
    ref = gpu_context(cfg, inp, stop_tol=tol)
    ref.run(100)
    k = ref.stats()["iters_last_run"]
    assert 1 < k < 100
    want = np.stack([ref.image(0, m) for m in range(cfg.nodes)])

    def calls(ctx, r):
        ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1, stop_tol=tol)
        ctx.run(100)

    ctxs, nr = run_world(cfg, inp, 2, 0, calls=calls)
    assert all(c.stats()["iters_last_run"] == k for c in ctxs)
    assert np.array_equal(node_images(ctxs, nr, cfg), want)


def test_profiling_phases():
    """tq_set_profiling: per-phase device times of the run (inner | encode | exchange | decode
    + dual) are positive where the phase has work, add up to the run's device time, and the
    iterates are bitwise those of the unprofiled run."""
    cfg = C.C4(1)
    inp = C.make_inputs(cfg, with_truth=False)
    a = gpu_context(cfg, inp)
    a.set_profiling(True)
    a.run(4)
    st = a.stats()
    b = gpu_context(cfg, inp)
    b.run(4)
    assert np.array_equal(a.image(0, 3), b.image(0, 3))
    assert st["phase_valid"] == 1
    inner, enc, exch, dual = st["phase_ms"]
    assert inner > 0 and enc > 0 and dual > 0 and exch >= 0
    assert inner > enc and inner > dual  # the projector-bound inner solves dominate
    assert abs(sum(st["phase_ms"]) - st["ms_last_run"]) <= 0.1 * st["ms_last_run"]
    assert b.stats()["phase_valid"] == 0


def test_node_bytes_graph_rule():
    """Graph rule (C2, ring, K-means 16): node i sends deg_i payloads and receives one from each
    neighbour; payload = 4K + 4 ceil(log2 K) ceil(n/32) bytes (R-17)."""
    cfg = C.C2()
    inp = C.make_inputs(cfg, with_truth=False)
    ctx = gpu_context(cfg, inp)
    ctx.run(1)
    pb = tomoq.payload_bytes(C.Q_KMEANS, cfg.k, cfg.N ** 2)
    assert pb == 4 * 16 + 4 * 4 * (cfg.N ** 2 // 32)
    for m in range(cfg.nodes):
        assert ctx.node_bytes(0, m) == (2 * pb, 2 * pb)
    assert sum(ctx.node_bytes(0, m)[0] for m in range(cfg.nodes)) == ctx.stats()["payload_bytes_logical"]


def test_node_bytes_paper_rule_matches_comm_model():
    """Paper rule, no quantizer: per node sent + received = Communication(M) = 2 (M-1)/M X
    (P:248-252), X = 4 N^2 bytes (fp32)."""
    cfg = C.C1()
    cfg.rule = C.RULE_PAPER
    inp = C.make_inputs(cfg, with_truth=False)
    ctx = gpu_context(cfg, inp)
    ctx.run(1)
    X = 4 * cfg.N ** 2
    for m in range(cfg.nodes):
        s, r = ctx.node_bytes(0, m)
        assert s + r == oracle.comm_model(cfg.nodes, X)
        assert s == r == (cfg.nodes - 1) * X // cfg.nodes


def test_node_bytes_entropy_coded():
    """Entropy-coded DCT payloads (NEXT-2) count their coded size: 16 + the oracle's JPEG
    stream length of the same coefficients, per neighbour."""
    cfg = C.scaled(C.C3(), 64, 96, iters=3)
    cfg.jpeg_restart = 4
    inp = C.make_inputs(cfg, with_truth=False)
    ctx = gpu_context(cfg, inp, precision=1)
    ctx.run(3)
    size = {}
    for m in range(cfg.nodes):
        x = ctx.export_state(0, m)[0].astype(np.float32).reshape(cfg.N, cfg.N)
        coef, _ = oracle.dct_encode(x, cfg.quality)
        size[m] = 16 + len(oracle.jpeg_encode(coef, 4))
    nb = {m: [] for m in range(cfg.nodes)}
    for i, j in inp.edges:
        nb[i].append(j)
        nb[j].append(i)
    for m in range(cfg.nodes):
        assert ctx.node_bytes(0, m) == (size[m] * len(nb[m]), sum(size[j] for j in nb[m]))

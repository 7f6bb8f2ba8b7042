"""Pins of the oracle's solvers and ADMM outer loop against dense linear algebra
(numpy.linalg on a brute-force system matrix), closed forms printed in / forced by
the paper, and invariants of the method."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2410_06106_b200 import synth
from tests.helpers import dense_joseph, rel

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def small_problem(N=16, n_ang=24, n_det=23, noise=0.01, seed=7):
    e = synth.random_ellipses(3, N, seed)
    d = synth.ellipse_sinogram(e, synth.default_angles(n_ang), n_det)
    return synth.add_noise(d, noise, seed + 1)


def test_cg_matches_dense_solve():
    """CG run for more steps than unknowns solves (A^T A + c I) x = A^T d + b' exactly
    (up to rounding): compare with a dense solve on the brute-force matrix."""
    N, n_ang, n_det = 16, 24, 23
    sel = list(range(1, n_ang, 3))
    A = dense_joseph(N, n_ang, n_det, sel)
    rng = np.random.default_rng(0)
    d = rng.standard_normal(len(sel) * n_det)
    bp = rng.standard_normal(N * N)
    c = 0.7
    x_ref = np.linalg.solve(A.T @ A + c * np.eye(N * N), A.T @ d + bp)
    x0 = rng.standard_normal((N, N))
    x = oracle.cg(d, bp, c, 400, x0, n_ang, sel)
    assert rel(x, x_ref) <= 1e-10


@pytest.mark.parametrize("e1", [1, 2, 5])
def test_cg_restructured_as_on_the_gpu_equals_oracle_cg(e1):
    """DESIGN.md R-8: the CUDA path runs CG with p.q formed as ||A p||^2 + c ||p||^2 from the
    forward projection, r -= alpha q fused into the backprojection, no backprojection in the
    last step, and the residual's A x kept across solves (A x += alpha A p).  Written out here
    with the oracle's projector on a dense problem, two consecutive solves (the second from
    the first's x with a new b', through the kept A x) equal the oracle's CG to fp64 rounding."""
    N, n_ang, n_det = 16, 24, 23
    sel = list(range(2, n_ang, 3))
    rng = np.random.default_rng(3 + e1)
    d = rng.standard_normal((len(sel), n_det))
    c = 1.3
    A = lambda v: oracle.project(v.reshape(N, N), n_ang, n_det, sel)
    At = lambda y: oracle.backproject(y, N, n_ang, sel).reshape(-1)

    def solve(x, bp, ax):
        r = At(d - ax) + bp - c * x
        p, rr = r.copy(), r @ r
        pp = rr
        for it in range(e1):
            s = A(p)
            alpha = rr / (np.sum(s * s) + c * pp)
            if it + 1 < e1:
                r = r - alpha * (At(s) + c * p)
                rr_new = r @ r
                beta = rr_new / rr
                rr = rr_new
            x = x + alpha * p
            ax = ax + alpha * s
            if it + 1 < e1:
                p = r + beta * p
                pp = p @ p
        return x, ax

    x = rng.standard_normal(N * N)
    bp1, bp2 = rng.standard_normal(N * N), rng.standard_normal(N * N)
    x1, ax1 = solve(x, bp1, A(x))
    x2, _ = solve(x1, bp2, ax1)
    o1 = oracle.cg(d, bp1, c, e1, x.reshape(N, N), n_ang, sel)
    o2 = oracle.cg(d, bp2, c, e1, o1, n_ang, sel)
    assert rel(x1, o1) <= 1e-12 and rel(x2, o2) <= 1e-12


def test_cg_one_step_is_exact_line_search():
    """One CG step from x0 is steepest descent with exact line search on the quadratic."""
    N, n_ang, n_det = 12, 10, 17
    sel = [0, 3, 7]
    A = dense_joseph(N, n_ang, n_det, sel)
    rng = np.random.default_rng(1)
    d, bp, x0 = rng.standard_normal(len(sel) * n_det), rng.standard_normal(N * N), rng.standard_normal(N * N)
    c = 2.0
    H = A.T @ A + c * np.eye(N * N)
    r = A.T @ d + bp - H @ x0
    x1 = x0 + (r @ r) / (r @ H @ r) * r
    assert rel(oracle.cg(d, bp, c, 1, x0.reshape(N, N), n_ang, sel), x1) <= 1e-12


def test_gd_one_step_from_zero():
    """Alg. 2 one step from u = 0: u = eta (A^T d + b')."""
    N, n_ang, n_det = 12, 10, 17
    sel = [1, 4, 5, 9]
    A = dense_joseph(N, n_ang, n_det, sel)
    rng = np.random.default_rng(2)
    d, bp = rng.standard_normal(len(sel) * n_det), rng.standard_normal(N * N)
    u = oracle.gd(d, bp, 0.3, 1e-3, 1, np.zeros((N, N)), n_ang, sel)
    assert rel(u, 1e-3 * (A.T @ d + bp)) <= 1e-13


def test_gd_converges_to_dense_solve():
    N, n_ang, n_det = 10, 8, 15
    sel = [0, 2, 5]
    A = dense_joseph(N, n_ang, n_det, sel)
    rng = np.random.default_rng(3)
    d, bp = rng.standard_normal(len(sel) * n_det), rng.standard_normal(N * N)
    c = 3.0
    H = A.T @ A + c * np.eye(N * N)
    x_ref = np.linalg.solve(H, A.T @ d + bp)
    eta = 1.0 / np.linalg.eigvalsh(H).max()
    u = oracle.gd(d, bp, c, eta, 3000, np.zeros((N, N)), n_ang, sel)
    assert rel(u, x_ref) <= 1e-9


def test_alg3_closed_form():
    """Alg. 3 with eta2 = 0.2, rho = 1, E2 = 10 from 0 toward the target
    u + lambda/rho = 1 gives 1 - 0.8^10 (scalar geometric contraction)."""
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))["alg3_contraction"]
    v = oracle.alg3(0.0, 1.0, 0.0, 1.0, 0.2, 10)
    assert abs(v - (1 - 0.8 ** 10)) < 1e-15
    assert abs(v - g["value"]) < 1e-9
    # the target u + lambda/rho is a fixed point for any E2
    assert abs(oracle.alg3(1.25, 1.0, 0.5, 2.0, 0.2, 37) - 1.25) < 1e-15


@pytest.fixture(scope="module")
def ls16():
    N, n_ang, n_det = 16, 24, 23
    d = small_problem(N, n_ang, n_det)
    A = dense_joseph(N, n_ang, n_det)
    x_ls = np.linalg.lstsq(A, d.ravel(), rcond=None)[0]
    return N, n_ang, n_det, d, A, x_ls


def test_graph_rule_converges_to_dense_least_squares(ls16):
    """North_star self-check: decentralized consensus ADMM over a ring of 4 nodes
    (round-robin angle split) converges to the centralized least-squares solution
    of eq:single_rec, computed densely by numpy.linalg.lstsq."""
    N, n_ang, n_det, d, A, x_ls = ls16
    o = oracle.OracleADMM(N, n_det, n_ang, 4, synth.ring(4), d, False, rule=0, inner=1, e1=20,
                          rho=0.1, threads=4)
    o.run(5000)
    assert rel(o.image(), x_ls) <= 1e-6
    # consensus: every node's private iterate agrees
    for i in range(4):
        assert rel(o.X[i], x_ls) <= 1e-5
    # invariant: sum_i alpha_i = 0 (edge terms cancel)
    assert np.linalg.norm(o.L.sum(axis=0)) <= 1e-12 * max(1.0, np.linalg.norm(o.L))


def test_paper_rule_single_node_is_proximal_point_to_ls(ls16):
    """M = 1 paper rule: x = conc(x[1]) = Alg. 3 output; the iteration is a proximal
    point method whose fixed point is the LS solution."""
    N, n_ang, n_det, d, A, x_ls = ls16
    o = oracle.OracleADMM(N, n_det, n_ang, 1, [], d, False, rule=1, inner=1, e1=20, rho=0.1,
                          e2=10, eta2=2.0)
    o.run(300)
    assert rel(o.image(), x_ls) <= 1e-8


def dense_paper_rule(A_blocks, d_blocks, M, N, rho, e2, eta2, iters):
    """eq:solve_u / eq:solve_x (Alg. 3) / eq:conc / eq:solve_lamda
    with the u-subproblem solved exactly by a dense solve."""
    n = N * N
    u = np.zeros((M, n)); lam = np.zeros((M, n)); x = np.zeros(n)
    rows = oracle.partition_rows(N, M) * N
    for _ in range(iters):
        for m in range(M):
            Am = A_blocks[m]
            u[m] = np.linalg.solve(Am.T @ Am + rho * np.eye(n), Am.T @ d_blocks[m] + rho * x - lam[m])
        xn = np.empty(n)
        for m in range(M):
            sl = slice(rows[m], rows[m + 1])
            xs = x[sl].copy()
            for _ in range(e2):
                xs = xs - eta2 * rho * (xs - u[m, sl] - lam[m, sl] / rho)
            xn[sl] = xs
        x = xn
        lam += rho * (u - x[None, :])
    return u, lam, x


def test_paper_rule_steps_match_dense_and_own_segment_dual_vanishes():
    N, n_ang, n_det, M = 16, 24, 23, 4
    d = small_problem(N, n_ang, n_det)
    off, idx = oracle.partition_angles(n_ang, M, False)
    Ab = [dense_joseph(N, n_ang, n_det, idx[off[m]:off[m + 1]]) for m in range(M)]
    db = [d[idx[off[m]:off[m + 1]]].ravel() for m in range(M)]
    rho = 0.5
    u, lam, x = dense_paper_rule(Ab, db, M, N, rho, 10, 0.2 / rho * 1.0, 3)
    o = oracle.OracleADMM(N, n_det, n_ang, M, [], d, False, rule=1, inner=1, e1=600, rho=rho,
                          e2=10, eta2=0.2 / rho)
    o.run(3)
    assert rel(o.X, u) <= 1e-9 and rel(o.XH[0], x) <= 1e-9 and rel(o.L, lam) <= 1e-9
    # E2 -> infinity with Q = identity: lambda_m vanishes on node m's own segment
    o2 = oracle.OracleADMM(N, n_det, n_ang, M, [], d, False, rule=1, inner=1, e1=10, rho=rho,
                           e2=400, eta2=1.0 / rho)
    o2.run(3)
    rows = oracle.partition_rows(N, M) * N
    for m in range(M):
        seg = o2.L[m, rows[m]:rows[m + 1]]
        assert np.max(np.abs(seg)) <= 1e-12 * max(1.0, np.max(np.abs(o2.L)))


def dense_consensus_rule(A_blocks, d_blocks, M, N, rho, iters):
    """The standard consensus ADMM of PAPER.md:121-131 (eq-compact:solve_u / solve_x /
    solve_lambda): u exact by a dense solve, x = mean over nodes of u + lambda/rho."""
    n = N * N
    u = np.zeros((M, n)); lam = np.zeros((M, n)); x = np.zeros(n)
    for _ in range(iters):
        for m in range(M):
            Am = A_blocks[m]
            u[m] = np.linalg.solve(Am.T @ Am + rho * np.eye(n), Am.T @ d_blocks[m] + rho * x - lam[m])
        x = (u + lam / rho).mean(axis=0)
        lam += rho * (u - x[None, :])
    return u, lam, x


def test_consensus_rule_steps_match_dense():
    """rule 2 (sharded consensus) step by step against the dense
    transcription of eq-compact:solve_u / solve_x / solve_lambda; Q = identity, so the
    sharding into segments does not change x."""
    N, n_ang, n_det, M = 16, 24, 23, 4
    d = small_problem(N, n_ang, n_det)
    off, idx = oracle.partition_angles(n_ang, M, False)
    Ab = [dense_joseph(N, n_ang, n_det, idx[off[m]:off[m + 1]]) for m in range(M)]
    db = [d[idx[off[m]:off[m + 1]]].ravel() for m in range(M)]
    rho = 0.5
    u, lam, x = dense_consensus_rule(Ab, db, M, N, rho, 3)
    o = oracle.OracleADMM(N, n_det, n_ang, M, [], d, False, rule=2, inner=1, e1=600, rho=rho)
    o.run(3)
    assert rel(o.X, u) <= 1e-9 and rel(o.XH[0], x) <= 1e-9 and rel(o.L, lam) <= 1e-9


def test_consensus_rule_converges_to_dense_least_squares(ls16):
    """Standard consensus ADMM converges to the centralized LS solution;
    with Q = identity sum_m lambda_m = 0 after every iteration (x is their mean)."""
    N, n_ang, n_det, d, A, x_ls = ls16
    o = oracle.OracleADMM(N, n_det, n_ang, 4, [], d, False, rule=2, inner=1, e1=20, rho=0.3, threads=4)
    o.run(4000)
    assert rel(o.image(), x_ls) <= 1e-5
    assert np.linalg.norm(o.L.sum(axis=0)) <= 1e-12 * max(1.0, np.linalg.norm(o.L))
    # M = 1: lambda stays 0 and x = u (a proximal point method, fixed point = LS)
    o1 = oracle.OracleADMM(N, n_det, n_ang, 1, [], d, False, rule=2, inner=1, e1=20, rho=0.1)
    o1.run(300)
    assert np.max(np.abs(o1.L)) == 0.0 and np.array_equal(o1.X[0], o1.XH[0])
    assert rel(o1.image(), x_ls) <= 1e-8


def test_admm_zero_data_stays_zero():
    N, n_ang, n_det = 16, 12, 23
    for rule in (0, 1, 2):
        for q in (0, 1, 2):
            o = oracle.OracleADMM(N, n_det, n_ang, 2, synth.ring(2), np.zeros((n_ang, n_det)), True,
                                  rule=rule, inner=1, e1=3, rho=1.0, qkind=q, K=4)
            o.run(3)
            assert not np.any(o.X) and not np.any(o.L) and not np.any(o.XH)


def test_admm_deterministic_and_thread_independent():
    N, n_ang, n_det = 16, 12, 23
    d = small_problem(N, n_ang, n_det)
    res = []
    for th in (1, 3):
        o = oracle.OracleADMM(N, n_det, n_ang, 4, synth.ring(4), d, True, rule=0, inner=1, e1=3,
                              rho=1.0, qkind=1, K=8, threads=th)
        o.run(4)
        res.append((o.X.copy(), o.L.copy(), o.XH.copy()))
    for a, b in zip(res[0], res[1]):
        assert np.array_equal(a, b)


def test_graph_rule_dual_sum_zero_with_quantizer():
    """The public value xhat_i is used at both ends of every edge, so sum_i alpha_i = 0
    holds exactly (up to rounding) even with a lossy Q."""
    N, n_ang, n_det = 16, 12, 23
    d = small_problem(N, n_ang, n_det)
    for q in (1, 2):
        o = oracle.OracleADMM(N, n_det, n_ang, 4, synth.ring(4), d, False, rule=0, inner=1, e1=3,
                              rho=1.0, qkind=q, K=8, quality=50)
        o.run(5)
        assert np.linalg.norm(o.L.sum(axis=0)) <= 1e-12 * max(1.0, np.linalg.norm(o.L))


def test_partitions_match_paper():
    g = json.load(open(os.path.join(GOLD, "paper_partitions.json")))
    off, idx = oracle.partition_angles(g["n_angles"], 10, False)
    assert list(np.diff(off)) == g["ten_nodes_counts"]
    f, l, s = g["ten_nodes_node0_first_last_step"]
    assert list(idx[off[0]:off[1]]) == list(range(f, l + 1, s))
    f, l, s = g["ten_nodes_node1_first_last_step"]
    assert list(idx[off[1]:off[2]]) == list(range(f, l + 1, s))
    off, idx = oracle.partition_angles(g["n_angles"], 2, False)
    assert list(np.diff(off)) == g["two_nodes_counts"]
    assert np.all(idx[off[0]:off[1]] % 2 == 0) and np.all(idx[off[1]:off[2]] % 2 == 1)
    off, idx = oracle.partition_angles(90, 4, True)
    assert list(np.diff(off)) == [23, 23, 22, 22] and list(idx) == list(range(90))
    assert list(oracle.partition_rows(12, 3)) == [0, 4, 8, 12]
    assert list(oracle.partition_rows(10, 3)) == [0, 4, 7, 10]


def test_cost_models():
    """PAPER.md:237 Memory(M) = D/M + 3X -> 3X; PAPER.md:250 Communication(M) =
    2(M-1)/M X -> 2X; SPEC.md:351 example D = X = 16 MB, M = 4 -> 52 MB."""
    MB = 2 ** 20
    assert oracle.memory_model(4, 16 * MB, 16 * MB) == 52 * MB
    assert oracle.memory_model(1, 5.0, 2.0) == 11.0
    assert abs(oracle.memory_model(10 ** 9, 1.0, 1.0) - 3.0) < 1e-8
    assert oracle.comm_model(1, 7.0) == 0.0
    assert oracle.comm_model(2, 7.0) == 7.0
    assert abs(oracle.comm_model(10 ** 9, 1.0) - 2.0) < 1e-8


def test_paper_rule_identity_bytes_match_comm_model():
    """With Q = identity each node sends its segment to the M-1 others: total sent per
    iteration = (M-1) X, i.e. per node (M-1)/M X sent and as much received, whose sum
    is Communication(M)."""
    N, n_ang, n_det, M = 16, 12, 23, 4
    o = oracle.OracleADMM(N, n_det, n_ang, M, [], small_problem(N, n_ang, n_det), False, rule=1,
                          inner=1, e1=2, rho=1.0)
    o.run(1)
    X = 4 * N * N
    assert o.bytes_per_iter == (M - 1) * X
    per_node_sent = o.bytes_per_iter / M
    assert per_node_sent * 2 == oracle.comm_model(M, X)


def dense_graph_rule(A_blocks, d_blocks, edges, M, N, rho, iters, K, lloyd, private_rhs=False):
    """Decentralized consensus ADMM over the graph (R-7) written out densely with
    the K-means quantizer on every exchanged iterate: the local problem solved
    exactly (dense solve), b'_i from the PUBLIC values xhat (R-11), alpha_i updated from the
    public values of node i and its neighbours."""
    n = N * N
    nb = [[] for _ in range(M)]
    for i, j in edges:
        nb[i].append(j)
        nb[j].append(i)
    x = np.zeros((M, n)); alpha = np.zeros((M, n)); xh = np.zeros((M, n))
    for _ in range(iters):
        for i in range(M):
            deg = len(nb[i])
            S = sum(xh[j] for j in nb[i])
            if private_rhs:  # the plausible mistake: the private iterates instead of xhat
                S = sum(x[j] for j in nb[i])
                bp = -alpha[i] + rho * (deg * x[i] + S)
            else:
                bp = -alpha[i] + rho * (deg * xh[i] + S)
            Ai = A_blocks[i]
            x[i] = np.linalg.solve(Ai.T @ Ai + 2 * rho * deg * np.eye(n), Ai.T @ d_blocks[i] + bp)
        for i in range(M):  # Q = Alg. 5 on the fp32 wire format (pinned in test_oracle_codecs)
            cen, lab = oracle.kmeans_encode(x[i].astype(np.float32), K, lloyd)
            xh[i] = oracle.kmeans_decode(cen, lab).astype(np.float64)
        for i in range(M):
            alpha[i] += rho * (len(nb[i]) * xh[i] - sum(xh[j] for j in nb[i]))
    return x, alpha, xh


def test_graph_rule_with_quantizer_steps_match_dense():
    """The graph rule with K-means (K = 8) step by step against its dense transcription: pins
    that b' and the dual use the quantized public values xhat, not the private x."""
    N, n_ang, n_det, M = 16, 24, 23, 4
    d = small_problem(N, n_ang, n_det)
    off, idx = oracle.partition_angles(n_ang, M, False)
    Ab = [dense_joseph(N, n_ang, n_det, idx[off[m]:off[m + 1]]) for m in range(M)]
    db = [d[idx[off[m]:off[m + 1]]].ravel() for m in range(M)]
    edges = synth.ring(M)
    x, alpha, xh = dense_graph_rule(Ab, db, edges, M, N, 0.5, 3, 8, 10)
    o = oracle.OracleADMM(N, n_det, n_ang, M, edges, d, False, rule=0, inner=1, e1=600, rho=0.5,
                          qkind=1, K=8, lloyd=10)
    o.run(3)
    assert rel(o.X, x) <= 1e-9 and rel(o.L, alpha) <= 1e-9
    assert np.array_equal(o.XH, xh)
    # b' from the private x instead of xhat (a plausible bug) gives a clearly different run
    x_bad, _, _ = dense_graph_rule(Ab, db, edges, M, N, 0.5, 3, 8, 10, private_rhs=True)
    assert rel(o.X, x_bad) > 1e-4


@pytest.mark.parametrize("rule", [0, 1, 2])
def test_stop_tol_first_iteration_below_tolerance(rule):
    """tq_params.stop_tol ("stopping criterion", R-13): the run stops after the first
    iteration k whose relative change ||x^{k+1} - x^k|| / ||x^{k+1}|| (max over the iterates:
    graph rule every node's x_i, paper / consensus rule x) is <= tol -- found here by running
    one iteration at a time and measuring the change with numpy."""
    N, n_ang, n_det = 16, 24, 23
    d = small_problem(N, n_ang, n_det)
    kw = dict(rule=rule, inner=1, e1=5, rho=1.0, e2=10, eta2=0.2)
    M = 4
    if rule == 1:  # the literal paper rule stalls for M > 1; M = 1 converges (prox point)
        M, kw["rho"], kw["eta2"] = 1, 0.1, 2.0
    edges = synth.ring(M) if M > 1 else []
    step = oracle.OracleADMM(N, n_det, n_ang, M, edges, d, False, **kw)
    tol = 2e-3
    k_stop = None
    for k in range(1, 300):
        prev = (step.X if rule == 0 else step.XH).copy()
        step.run(1)
        cur = step.X if rule == 0 else step.XH
        r = max(np.linalg.norm(cur[i] - prev[i]) / np.linalg.norm(cur[i]) for i in range(len(cur)))
        if r <= tol:
            k_stop = k
            break
    assert k_stop is not None and k_stop > 2
    o = oracle.OracleADMM(N, n_det, n_ang, M, edges, d, False, stop_tol=tol, **kw)
    o.run(300)
    assert o.last_run_iters == k_stop and o.iters == k_stop
    assert o.last_change <= tol
    assert np.array_equal(o.X, step.X) and np.array_equal(o.XH, step.XH)
    # stop_tol = 0: the requested count
    o0 = oracle.OracleADMM(N, n_det, n_ang, M, edges, d, False, **kw)
    o0.run(7)
    assert o0.last_run_iters == 7


def test_stop_tol_zero_data_stops_after_one_iteration():
    """Zero data: x stays 0, the change 0/0 counts as 0, so the run stops after iteration 1."""
    N, n_ang, n_det = 16, 12, 23
    o = oracle.OracleADMM(N, n_det, n_ang, 2, synth.ring(2), np.zeros((n_ang, n_det)), True,
                          rule=0, inner=1, e1=3, rho=1.0, stop_tol=1e-6)
    o.run(50)
    assert o.last_run_iters == 1 and o.last_change == 0.0

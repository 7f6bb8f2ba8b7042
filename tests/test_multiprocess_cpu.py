"""N > 1 path on the CPU: two processes (torch.distributed, gloo, world size 2) run the
graph-rule ADMM of DESIGN.md R-7 with the ADMM nodes split over the ranks exactly as
libtomoq places them (node i on rank i mod world), moving each iteration's
quantized public values x_hat along the cross-rank edges with point-to-point
send/recv in the order libtomoq's exchange plan (tq_exchange_plan) prescribes.
The result must equal the single-process oracle run bit for bit: the plan delivers
every neighbour payload a rank needs, both ends post matching sequences (no
deadlock), and the exchange only moves bytes."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2410_06106_b200 import configs as C
from paper_2410_06106_b200 import synth, tomoq


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    cfg = C.scaled(C.C2(), 32, 36, nodes=4, k=8, lloyd=5)
    return cfg, C.make_inputs(cfg, with_truth=False)


def _distributed_admm(rank, world, port, iters, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, inp = _case()
        M, N = cfg.nodes, cfg.N
        n = N * N
        off, idx = oracle.partition_angles(cfg.n_angles, M, cfg.split == C.SPLIT_CONTIG)
        sino = inp.sino[0].astype(np.float64)
        adj = [[] for _ in range(M)]
        for i, j in inp.edges:  # neighbour order = the oracle's adjacency order
            adj[i].append(j)
            adj[j].append(i)
        sends, recvs = tomoq.exchange_plan(M, inp.edges, tomoq.RULE_GRAPH, rank, world)
        mine = [i for i in range(M) if i % world == rank]
        X = {i: np.zeros(n) for i in mine}
        A = {i: np.zeros(n) for i in mine}
        XH = {}  # public values this rank knows (own + received)
        for i in range(M):
            if i in mine or any(nd == i for nd, _ in recvs):
                XH[i] = np.zeros(n)
        rho = cfg.rho
        for _ in range(iters):
            for i in mine:
                deg = len(adj[i])
                S = np.zeros(n)
                for j in adj[i]:
                    S = S + XH[j]
                bp = -A[i] + rho * (deg * XH[i] + S)
                sel = idx[off[i]:off[i + 1]]
                d = sino[sel]
                X[i] = oracle.cg(d, bp.reshape(N, N), 2.0 * rho * deg, cfg.e1, X[i].reshape(N, N),
                                 cfg.n_angles, sel).ravel()
            for i in mine:
                cen, lab = oracle.kmeans_encode(X[i].astype(np.float32), cfg.k, cfg.lloyd)
                XH[i] = oracle.kmeans_decode(cen, lab).astype(np.float64)
            # the exchange, in plan order: all sends and receives of the iteration
            reqs = []
            for node, peer in sends:
                reqs.append(dist.isend(torch.from_numpy(XH[node].copy()), dst=peer))
            bufs = []
            for node, peer in recvs:
                b = torch.empty(n, dtype=torch.float64)
                reqs.append(dist.irecv(b, src=peer))
                bufs.append((node, b))
            for r in reqs:
                r.wait()
            for node, b in bufs:
                XH[node] = b.numpy().copy()
            for i in mine:
                deg = len(adj[i])
                S = np.zeros(n)
                for j in adj[i]:
                    S = S + XH[j]
                A[i] = A[i] + rho * (deg * XH[i] - S)
        np.save(os.path.join(out, f"x_rank{rank}.npy"), np.stack([X[i] for i in mine]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_matches_single_process(tmp_path):
    iters = 3
    world = 2
    port = _free_port()
    mp.start_processes(_distributed_admm, args=(world, port, iters, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    cfg, inp = _case()
    ref = oracle.OracleADMM(cfg.N, cfg.n_det, cfg.n_angles, cfg.nodes, inp.edges,
                            inp.sino[0].astype(np.float64), cfg.split == C.SPLIT_CONTIG, rule=0,
                            inner=1, e1=cfg.e1, rho=cfg.rho, qkind=1, K=cfg.k, lloyd=cfg.lloyd,
                            threads=1).run(iters)
    for r in range(world):
        got = np.load(os.path.join(tmp_path, f"x_rank{r}.npy"))
        nodes = [i for i in range(cfg.nodes) if i % world == r]
        for k, i in enumerate(nodes):
            np.testing.assert_allclose(got[k], ref.X[i], rtol=0, atol=1e-12 * np.abs(ref.X[i]).max())
    assert np.abs(ref.X).max() > 0


def _distributed_consensus(rank, world, port, iters, out):
    """Rule 2 (P:121-131 with x sharded in segments) split over the ranks as libtomoq
    places it: per-rank partial sums of u + lambda/rho, one reduce per segment onto the
    rank owning that segment (Ctx::reduce_sums), x[m] formed there, then the all-gather
    of the segments in tq_exchange_plan order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, inp = _case()
        M, N = cfg.nodes, cfg.N
        n = N * N
        off, idx = oracle.partition_angles(cfg.n_angles, M, cfg.split == C.SPLIT_CONTIG)
        rows = [m * N // M for m in range(M + 1)]  # the oracle's row partition (M | N here)
        sino = inp.sino[0].astype(np.float64)
        sends, recvs = tomoq.exchange_plan(M, inp.edges, tomoq.RULE_CONSENSUS, rank, world)
        mine = [i for i in range(M) if i % world == rank]
        X = {i: np.zeros(n) for i in mine}
        A = {i: np.zeros(n) for i in mine}
        x = np.zeros(n)
        rho = cfg.rho
        for _ in range(iters):
            for i in mine:
                sel = idx[off[i]:off[i + 1]]
                X[i] = oracle.cg(sino[sel], (rho * x - A[i]).reshape(N, N), rho, cfg.e1,
                                 X[i].reshape(N, N), cfg.n_angles, sel).ravel()
            psum = np.zeros(n)
            for i in mine:
                psum = psum + (X[i] + A[i] / rho)
            t = torch.from_numpy(psum)
            for m in range(M):
                seg = t[rows[m] * N:rows[m + 1] * N].clone()
                dist.reduce(seg, dst=m % world)
                if m % world == rank:
                    x[rows[m] * N:rows[m + 1] * N] = seg.numpy() / M
            reqs, bufs = [], []
            for node, peer in sends:
                reqs.append(dist.isend(torch.from_numpy(x[rows[node] * N:rows[node + 1] * N].copy()), dst=peer))
            for node, peer in recvs:
                b = torch.empty((rows[node + 1] - rows[node]) * N, dtype=torch.float64)
                reqs.append(dist.irecv(b, src=peer))
                bufs.append((node, b))
            for r in reqs:
                r.wait()
            for node, b in bufs:
                x[rows[node] * N:rows[node + 1] * N] = b.numpy()
            for i in mine:
                A[i] = A[i] + rho * (X[i] - x)
        np.save(os.path.join(out, f"x_rank{rank}.npy"), x)
        np.save(os.path.join(out, f"u_rank{rank}.npy"), np.stack([X[i] for i in mine]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_consensus_rule_matches_single_process(tmp_path):
    iters = 3
    world = 2
    port = _free_port()
    mp.start_processes(_distributed_consensus, args=(world, port, iters, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    cfg, inp = _case()
    ref = oracle.OracleADMM(cfg.N, cfg.n_det, cfg.n_angles, cfg.nodes, inp.edges,
                            inp.sino[0].astype(np.float64), cfg.split == C.SPLIT_CONTIG, rule=2,
                            inner=1, e1=cfg.e1, rho=cfg.rho, qkind=0, threads=1).run(iters)
    # the cross-rank sum order differs from the oracle's node order: equal to rounding
    for r in range(world):
        x = np.load(os.path.join(tmp_path, f"x_rank{r}.npy"))
        np.testing.assert_allclose(x, ref.XH[0], rtol=0, atol=1e-11 * np.abs(ref.XH[0]).max())
        got = np.load(os.path.join(tmp_path, f"u_rank{r}.npy"))
        for k, i in enumerate(i for i in range(cfg.nodes) if i % world == r):
            np.testing.assert_allclose(got[k], ref.X[i], rtol=0, atol=1e-11 * np.abs(ref.X[i]).max())
    assert np.abs(ref.XH[0]).max() > 0

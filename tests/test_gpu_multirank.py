"""world > 1 on one GPU: several ranks of one world as contexts of this process (one host
thread per rank) over the in-process loopback transport (tq_loopback_id, include/tomoq.h).

The loopback runs the same exchange plan, payload buffers and per-iteration graph
segmentation (inner solves | [segment reduce] | encode | exchange | decode + dual) as the
NCCL path; only the byte movement differs.  SURVEY.md 8(c) parity item 5: the exchange moves
bytes and every reduction is fixed-order per node, so a run split over `world` ranks equals
the world == 1 run bit for bit (graph and paper rules).  The consensus rule's cross-rank
segment sum changes the fp64 summation order (R-24): equal to fp64 rounding.

PAPER.md:188 (the segment exchange is "the primary bandwidth demand"), :248-252
(per-node communication)."""
import threading

import numpy as np
import pytest

from paper_2410_06106_b200 import configs as C
from paper_2410_06106_b200 import tomoq
from tests.cases import gpu_context, rel

pytestmark = pytest.mark.gpu


def run_world(cfg, inp, world, iters, precision=0, node_rank=None, calls=None):
    """Run `iters` iterations of cfg split over `world` loopback ranks; returns the per-rank
    contexts (still open) and the node -> rank map.  `calls(ctx, rank)` replaces the plain run."""
    lid = tomoq.loopback_id()
    nr = list(node_rank) if node_rank is not None else [m % world for m in range(cfg.nodes)]
    ctxs, errs = [None] * world, []

    def worker(r):
        try:
            ctx = tomoq.Context(cfg.N, cfg.n_angles, cfg.n_det, cfg.nodes, inp.edges, split=cfg.split,
                                rule=cfg.rule, n_slices=len(inp.sino), rank=r, world=world, nccl_id=lid,
                                precision=precision, node_rank=nr, projector=cfg.projector)
            ctxs[r] = ctx
            ctx.set_params(cfg.rho, inner=cfg.inner, e1=cfg.e1, e2=cfg.e2, eta2=cfg.eta2)
            ctx.set_quantizer(cfg.quant, k=cfg.k, lloyd=cfg.lloyd, quality=cfg.quality,
                              jpeg_restart=cfg.jpeg_restart)
            for s, d in enumerate(inp.sino):
                ctx.set_sinogram(s, d)
            if calls is None:
                ctx.run(iters)
            else:
                calls(ctx, r)
        except Exception as e:  # reported by the main thread
            errs.append((r, e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a rank hung"
    assert not errs, errs
    return ctxs, nr


def node_images(ctxs, nr, cfg, s=0):
    return np.stack([ctxs[nr[m]].image(s, m) for m in range(cfg.nodes)])


def reference_images(cfg, inp, iters, precision=0, s_list=(0,)):
    ctx = gpu_context(cfg, inp, precision=precision)
    ctx.run(iters)
    out = {s: np.stack([ctx.image(s, m) for m in range(cfg.nodes)]) for s in s_list}
    ctx.close()
    return out


def close_all(ctxs):
    for c in ctxs:
        if c is not None:
            c.close()


@pytest.mark.parametrize("world", [2, 4])
def test_graph_rule_c2_bitwise(world):
    """Config 2 as stated (256^2, ring of 8, K-means 16): world 2 / 4 == world 1, bit for bit."""
    cfg = C.C2()
    inp = C.make_inputs(cfg, with_truth=False)
    iters = 6
    ref = reference_images(cfg, inp, iters)[0]
    ctxs, nr = run_world(cfg, inp, world, iters)
    got = node_images(ctxs, nr, cfg)
    st = [c.stats() for c in ctxs]
    close_all(ctxs)
    assert np.array_equal(got, ref)
    # every rank moved bytes across the transport (interleaved map: every ring edge crosses ranks)
    for s in st:
        assert s["world"] == world and s["nccl_bytes_sent"] > 0 and s["nccl_bytes_recv"] > 0


@pytest.mark.parametrize("world", [2, 4, 8])
def test_graph_rule_bench_config_bitwise(world):
    """The bench workload C4_G1 (1024^2, 8 nodes on a random 4-regular graph, K-means 64)
    split over 2 / 4 / 8 ranks (8: one node per rank, the layout of an 8-GPU run) equals the
    one-rank run bit for bit."""
    cfg = C.C4(1)
    inp = C.make_inputs(cfg, with_truth=False)
    iters = 2
    ref = reference_images(cfg, inp, iters)[0]
    ctxs, nr = run_world(cfg, inp, world, iters)
    got = node_images(ctxs, nr, cfg)
    close_all(ctxs)
    assert np.array_equal(got, ref)


def test_graph_rule_kept_ax_refresh_cadence_bitwise():
    """20 iterations (past the kept A x's refresh at iteration 16, R-8): one rank runs them as
    four-iteration graphs, two ranks one iteration per graph between exchanges -- the refresh
    points coincide and the runs stay bitwise equal."""
    cfg = C.C2()
    inp = C.make_inputs(cfg, with_truth=False)
    iters = 20
    ref = reference_images(cfg, inp, iters)[0]
    ctxs, nr = run_world(cfg, inp, 2, iters)
    got = node_images(ctxs, nr, cfg)
    close_all(ctxs)
    assert np.array_equal(got, ref)


def test_graph_rule_contiguous_map_and_uneven_ranks():
    """A non-interleaved node -> rank map with unequal node counts (3 ranks: 4 + 3 + 1 nodes)."""
    cfg = C.C2()
    inp = C.make_inputs(cfg, with_truth=False)
    iters = 4
    ref = reference_images(cfg, inp, iters)[0]
    ctxs, nr = run_world(cfg, inp, 3, iters, node_rank=[0, 0, 0, 0, 1, 1, 1, 2])
    got = node_images(ctxs, nr, cfg)
    close_all(ctxs)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("jpeg_restart", [0, 4])
def test_graph_rule_dct_torus_bitwise(jpeg_restart):
    """Config 3's structure (4x4 torus of 16 nodes, DCT q50) at 128^2 over 4 ranks, with plain
    and entropy-coded (JPEG, R-25) payloads: the full payload capacity crosses ranks."""
    cfg = C.scaled(C.C3(), 128, 192, iters=5)
    cfg.jpeg_restart = jpeg_restart
    inp = C.make_inputs(cfg, with_truth=False)
    ref = reference_images(cfg, inp, cfg.iters)[0]
    ctxs, nr = run_world(cfg, inp, 4, cfg.iters)
    got = node_images(ctxs, nr, cfg)
    close_all(ctxs)
    assert np.array_equal(got, ref)


def test_graph_rule_two_slices_alternating_codecs():
    """Config 5's structure (complete graph of 8, slice 0 K-means 32, slice 1 DCT q75) at 64^2,
    two slices over 2 ranks."""
    cfg = C.scaled(C.C5(slices=2), 64, 96, iters=4)
    inp = C.make_inputs(cfg, with_truth=False)
    ref = reference_images(cfg, inp, cfg.iters, s_list=(0, 1))
    ctxs, nr = run_world(cfg, inp, 2, cfg.iters)
    for s in (0, 1):
        assert np.array_equal(node_images(ctxs, nr, cfg, s), ref[s])
    close_all(ctxs)


@pytest.mark.parametrize("quant", [C.Q_NONE, C.Q_KMEANS, C.Q_DCT])
@pytest.mark.parametrize("world", [2, 4])
def test_paper_rule_bitwise(quant, world):
    """The paper's segment rule (the all-gather of P:188 over the same send/recv
    plan) on config 1 (4 nodes, 16-row segments), unquantized and quantized."""
    cfg = C.C1()
    cfg.rule, cfg.quant, cfg.k, cfg.iters = C.RULE_PAPER, quant, 8, 6
    inp = C.make_inputs(cfg, with_truth=False)
    ref = reference_images(cfg, inp, cfg.iters)[0]
    ctxs, nr = run_world(cfg, inp, world, cfg.iters)
    got = node_images(ctxs, nr, cfg)
    xg = [c.image(0, -1) for c in ctxs]  # the consensus x: identical on every rank
    close_all(ctxs)
    assert np.array_equal(got, ref)
    for x in xg[1:]:
        assert np.array_equal(x, xg[0])


@pytest.mark.parametrize("quant", [C.Q_NONE, C.Q_KMEANS])
def test_consensus_rule_segment_reduce(quant):
    """The consensus rule's per-segment sum across ranks (R-24): fp64 verification mode,
    world 2 equals world 1 to fp64 rounding of the changed summation order."""
    cfg = C.C1()
    cfg.rule, cfg.quant, cfg.k, cfg.iters = C.RULE_CONSENSUS, quant, 8, 6
    inp = C.make_inputs(cfg, with_truth=False)
    ref = reference_images(cfg, inp, cfg.iters, precision=1)[0]
    ctxs, nr = run_world(cfg, inp, 2, cfg.iters, precision=1)
    got = node_images(ctxs, nr, cfg)
    close_all(ctxs)
    assert rel(got, ref) <= 1e-10


def test_loopback_async_api_sequence():
    """The asynchronous API sequence of bench.py's e2e loop on every rank (set_sinogram,
    run_async, image_async, wait) equals the blocking world == 1 sequence."""
    import torch
    cfg = C.C2()
    inp = C.make_inputs(cfg, with_truth=False)
    ref = reference_images(cfg, inp, 3)[0]
    outs = {}

    def calls(ctx, r):
        st = torch.cuda.Stream()
        cp = torch.cuda.Stream()
        bufs = [torch.empty(cfg.N * cfg.N, dtype=torch.float32).pin_memory() for _ in range(2)]
        for k in range(3):
            ctx.set_sinogram(0, inp.sino[0])
            ctx.run_async(1, st)
            ctx.image_async(bufs[k & 1], cp, 0, r)
        ctx.wait()
        cp.synchronize()
        outs[r] = bufs[0].numpy().copy()  # iteration 3 went to buffer 0

    ctxs, nr = run_world(cfg, inp, 2, 0, calls=calls)
    close_all(ctxs)
    for r in (0, 1):
        assert np.array_equal(outs[r].reshape(cfg.N, cfg.N), ref[r])


def test_loopback_peer_failure_times_out(monkeypatch):
    """A rank that never reaches the exchange makes its peers fail with TQ_ENCCL after
    TQ_LOOPBACK_TIMEOUT_S seconds instead of hanging."""
    monkeypatch.setenv("TQ_LOOPBACK_TIMEOUT_S", "3")
    cfg = C.C1()
    inp = C.make_inputs(cfg, with_truth=False)

    def calls(ctx, r):
        if r == 1:
            raise RuntimeError("rank 1 stops")
        ctx.run(1)

    with pytest.raises(AssertionError) as e:
        run_world(cfg, inp, 2, 1, calls=calls)
    msg = str(e.value)
    assert "rank 1 stops" in msg and "TQ_ENCCL" in msg and "timed out" in msg

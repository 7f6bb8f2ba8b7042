"""Node groups (DESIGN.md 6.1 "node groups"): the graph rule's fp32 CG + K-means stages run as
concurrent launch chains over contiguous node ranges (default for N >= 512: one per node, up to 8).  Every kernel's result for a
node depends only on that node's inputs and per-node fixed-order reductions, so the grouped
iteration must equal the single-chain one (TQ_GROUPS=1) bit for bit: x_i, alpha_i, the decoded
x_hat_i and the K-means labels of every node (Alg. 4)."""
from dataclasses import replace

import numpy as np
import pytest

from paper_2410_06106_b200 import configs as C
from tests.cases import export_all, gpu_context

pytestmark = pytest.mark.gpu


def _run(cfg, inp, iters, groups, monkeypatch, keep_labels=False):
    monkeypatch.setenv("TQ_GROUPS", str(groups))
    ctx = gpu_context(cfg, inp, keep_labels=keep_labels)
    ctx.run(iters)
    st = ctx.stats()
    X, Lm, XH = export_all(ctx, cfg)
    labels = [ctx.labels(0, m, cfg.N * cfg.N) for m in range(cfg.nodes)] if keep_labels else None
    ctx.close()
    return st, X, Lm, XH, labels


def _same(a, b):
    for u, v in zip(a[1:4], b[1:4]):
        np.testing.assert_array_equal(u, v)


@pytest.mark.parametrize("name,cfg,iters", [
    ("C1 unquantized, 4 nodes", C.C1(), 6),
    ("C2 K-means 16, 8 nodes", C.C2(), 4),
    ("C2 on 7 nodes (groups 3 + 4)", replace(C.C2(), nodes=7, graph="ring"), 4),
    ("C4_G1 bench workload", C.C4(1), 3),
    ("C2 with the Siddon projector (R-26)", replace(C.C2(), projector=1), 4),
])
def test_groups_bitwise_equal_to_one_chain(name, cfg, iters, monkeypatch):
    inp = C.make_inputs(cfg, with_truth=False)
    one = _run(cfg, inp, iters, 1, monkeypatch)
    two = _run(cfg, inp, iters, 2, monkeypatch)
    assert one[0]["node_groups"] == 1 and two[0]["node_groups"] == 2, name
    _same(one, two)


@pytest.mark.parametrize("groups", [3, 4])
def test_more_groups_bitwise_equal(groups, monkeypatch):
    """Uneven contiguous ranges: 7 nodes as 2 + 2 + 3 / 1 + 2 + 2 + 2."""
    cfg = replace(C.C2(), nodes=7, graph="ring")
    inp = C.make_inputs(cfg, with_truth=False)
    one = _run(cfg, inp, 3, 1, monkeypatch)
    many = _run(cfg, inp, 3, groups, monkeypatch)
    assert many[0]["node_groups"] == groups
    _same(one, many)


def test_default_groups(monkeypatch):
    """Default: one group per node (up to 8) for N >= 512, one chain below."""
    monkeypatch.delenv("TQ_GROUPS", raising=False)
    for cfg, want in ((C.C4(1), 8), (C.C2(), 1)):
        inp = C.make_inputs(cfg, with_truth=False)
        ctx = gpu_context(cfg, inp)
        ctx.run(1)
        assert ctx.stats()["node_groups"] == want, cfg.name
        ctx.close()


@pytest.mark.parametrize("groups", [8])
def test_one_group_per_node_bitwise_c4(groups, monkeypatch):
    cfg = C.C4(1)
    inp = C.make_inputs(cfg, with_truth=False)
    one = _run(cfg, inp, 3, 1, monkeypatch)
    many = _run(cfg, inp, 3, groups, monkeypatch)
    assert many[0]["node_groups"] == groups
    _same(one, many)


def test_groups_residual_projection_every_solve(monkeypatch):
    """TQ_AX_MAXAGE=0: each group's solve starts from the forward-projected residual d - A x
    (the group's rows of the band reduction with the data term) instead of the kept A x."""
    monkeypatch.setenv("TQ_AX_MAXAGE", "0")
    cfg = C.C2()
    inp = C.make_inputs(cfg, with_truth=False)
    one = _run(cfg, inp, 4, 1, monkeypatch)
    many = _run(cfg, inp, 4, 4, monkeypatch)
    assert many[0]["node_groups"] == 4
    _same(one, many)


def test_groups_labels_and_kept_ax_refresh(monkeypatch):
    """K-means labels, and enough iterations to pass the kept A x refresh (TQ_AX_MAXAGE)."""
    monkeypatch.setenv("TQ_AX_MAXAGE", "3")
    cfg = C.C2()
    inp = C.make_inputs(cfg, with_truth=False)
    one = _run(cfg, inp, 8, 1, monkeypatch, keep_labels=True)
    two = _run(cfg, inp, 8, 2, monkeypatch, keep_labels=True)
    assert two[0]["node_groups"] == 2
    _same(one, two)
    for a, b in zip(one[4], two[4]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("name,cfg,groups", [
    ("C3 DCT q50, 16 nodes torus", C.C3(), 8),
    ("C3 DCT q50, 16 nodes torus, 3 groups", C.C3(), 3),
    ("two C2 slices, K-means / DCT alternating", replace(C.C2(), quant=C.Q_ALT, quality=75, slices=2), 4),
    ("C3 JPEG entropy-coded DCT, restart 4", replace(C.C3(), jpeg_restart=4), 8),
    ("C3 JPEG entropy-coded DCT, restart 1, 3 groups", replace(C.C3(), jpeg_restart=1), 3),
])
def test_groups_dct_and_alternating_bitwise(name, cfg, groups, monkeypatch):
    """Plain DCT payloads and slices alternating K-means / DCT (C5's codec mix): each group encodes
    its contiguous subrange of each codec's batch."""
    inp = C.make_inputs(cfg, with_truth=False)
    one = _run_slices(cfg, inp, 3, 1, monkeypatch)
    many = _run_slices(cfg, inp, 3, groups, monkeypatch)
    assert one[0]["node_groups"] == 1 and many[0]["node_groups"] == groups, name
    # the coded payload sizes (JPEG: gathered from the groups' coders) are the same bytes
    assert one[0]["payload_bytes_logical"] == many[0]["payload_bytes_logical"], name
    for a, b in zip(one[1], many[1]):
        np.testing.assert_array_equal(a, b)


def _run_slices(cfg, inp, iters, groups, monkeypatch):
    monkeypatch.setenv("TQ_GROUPS", str(groups))
    ctx = gpu_context(cfg, inp)
    ctx.run(iters)
    st = ctx.stats()
    out = [np.concatenate(export_all(ctx, cfg, s)) for s in range(len(inp.sino))]
    ctx.close()
    return st, out


def test_groups_not_used_where_not_applicable(monkeypatch):
    """fp64 and GD keep the single chain (tq_stats says so)."""
    monkeypatch.setenv("TQ_GROUPS", "2")
    for cfg, prec in ((C.C2(), 1), (replace(C.C2(), inner=C.INNER_GD, e1=10), 0)):
        inp = C.make_inputs(cfg, with_truth=False)
        ctx = gpu_context(cfg, inp, precision=prec)
        ctx.run(1)
        assert ctx.stats()["node_groups"] == 1, (cfg.name, prec, cfg.inner)
        ctx.close()

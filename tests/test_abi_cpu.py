"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every
symbol include/tomoq.h declares, and its host-side logic (angle partition of
PAPER.md:319-320, exchange plans, payload sizes, argument validation) is right.
No compute call is made here."""
import json
import os
import re

import numpy as np
import pytest

from paper_2410_06106_b200 import synth, tomoq

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2410_06106_b200 import build
    build.build()


def header_functions():
    src = open(tomoq.HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tq_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = tomoq.lib()
    names = header_functions()
    assert len(names) >= 24
    for n in names:
        assert hasattr(L, n), n


def test_partition_matches_paper():
    g = json.load(open(os.path.join(GOLD, "paper_partitions.json")))
    off, idx = tomoq.partition_angles(804, 10, tomoq.SPLIT_RR)
    assert list(np.diff(off)) == g["ten_nodes_counts"]
    assert list(idx[off[1]:off[2]]) == list(range(1, 802, 10))
    off, idx = tomoq.partition_angles(90, 4, tomoq.SPLIT_CONTIG)
    assert list(np.diff(off)) == [23, 23, 22, 22]


def test_payload_bytes():
    # C2: 256^2 values, K = 16 -> 64 B centres + 4 bit-planes of 2048 words
    assert tomoq.payload_bytes(tomoq.Q_KMEANS, 16, 65536) == 32832
    assert tomoq.payload_bytes(tomoq.Q_KMEANS, 64, 1 << 20) == 786688
    assert tomoq.payload_bytes(tomoq.Q_DCT, 50, 512 * 512) == 524296
    assert tomoq.payload_bytes(tomoq.Q_NONE, 0, 100, 1) == 800


@pytest.mark.parametrize("kind,M,world", [("ring", 8, 2), ("ring", 8, 4), ("torus", 16, 8),
                                          ("regular4", 16, 8), ("complete", 8, 8), ("ring", 2, 2)])
@pytest.mark.parametrize("rule", [tomoq.RULE_GRAPH, tomoq.RULE_PAPER, tomoq.RULE_CONSENSUS])
def test_exchange_plans_pair_up(kind, M, world, rule):
    edges = synth.make_graph(kind, M, 4003)
    plans = [tomoq.exchange_plan(M, edges, rule, r, world) for r in range(world)]
    owner = [i % world for i in range(M)]
    for a in range(world):
        sends = plans[a][0]
        for b in range(world):
            sa = [n for (n, p) in sends if p == b]
            rb = [n for (n, p) in plans[b][1] if p == a]
            assert sa == rb  # same payloads, same order (matched NCCL p2p sequences)
            assert all(owner[n] == a for n in sa)
    # graph rule: every cross-rank neighbour payload arrives exactly once per rank
    if rule == tomoq.RULE_GRAPH:
        for r in range(world):
            need = {j for (i, j) in edges if owner[i] == r and owner[j] != r} | \
                   {i for (i, j) in edges if owner[j] == r and owner[i] != r}
            got = [n for (n, _) in plans[r][1]]
            assert sorted(got) == sorted(need)
    else:
        for r in range(world):
            got = sorted(n for (n, _) in plans[r][1])
            assert got == sorted(n for n in range(M) if owner[n] != r)


def test_create_validates_geometry():
    with pytest.raises(tomoq.TomoQError) as e:
        tomoq.Context(60, 90, 91, 4, synth.ring(4))   # N not a multiple of 8
    assert e.value.code == 1
    with pytest.raises(tomoq.TomoQError) as e:
        tomoq.Context(64, 90, 89, 4, synth.ring(4))   # n_det < N sqrt 2
    assert e.value.code == 1 and "n_det" in str(e.value)
    with pytest.raises(tomoq.TomoQError):
        tomoq.Context(64, 90, 91, 4, [(0, 1), (2, 3)])  # disconnected graph
    with pytest.raises(tomoq.TomoQError):
        tomoq.Context(64, 90, 91, 4, [(0, 0)])          # self loop

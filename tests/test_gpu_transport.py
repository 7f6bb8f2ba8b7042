"""The exchange layer alone (row A7; PAPER.md:188 "the primary bandwidth demand", :248-252 the
per-node communication), through tq_debug_transport_check (include/tomoq.h).

The engine's world > 1 runs are covered over the in-process loopback (test_gpu_multirank.py).
NCCL refuses two ranks on one GPU ("Duplicate GPU detected", profiles/r2_nccl_duplicate_gpu.txt)
and the pool's boxes have one B200, so the NCCL transport is executed here at world == 1 with
every rank sending to itself: the same NcclTransport code the engine calls at world > 1
(ncclCommInitRank, ncclSend / ncclRecv in one group, the grouped per-segment ncclReduce,
ncclAllReduce for the stop test).  Expected values are exact and computed on the host."""
import threading

import pytest

from paper_2410_06106_b200 import tomoq

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nbytes,n_doubles", [(1, 1), (4099, 1000), (1 << 22, 1 << 18)])
def test_nccl_transport_world1_self_exchange(nbytes, n_doubles):
    tid = tomoq.nccl_unique_id()
    tomoq.debug_transport_check(tid, 0, 1, 0, nbytes=nbytes, n_doubles=n_doubles, rounds=3)


def _loopback_world(world, nbytes, n_doubles):
    tid = tomoq.loopback_id()
    errs = []

    def worker(r):
        try:
            tomoq.debug_transport_check(tid, r, world, 0, nbytes=nbytes, n_doubles=n_doubles, rounds=3)
        except Exception as e:
            errs.append((r, e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "a rank hung"
    assert not errs, errs


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_loopback_transport_check(world):
    _loopback_world(world, 12345, 4097)


def test_transport_check_rejects_bad_arguments():
    tid = tomoq.loopback_id()
    with pytest.raises(Exception):
        tomoq.debug_transport_check(tid, 0, 1, 0, nbytes=0)
    with pytest.raises(Exception):
        tomoq.debug_transport_check(tid, 1, 1, 0)

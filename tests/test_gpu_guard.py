"""Out-of-bounds writes and reads of never-written device memory, without compute-sanitizer
(closed on the GPU pool): tools/guard_run.py runs every kernel family plainly and under
TQ_GUARD=1 (include/tomoq.h tq_debug_guard_check: 256-byte guard bands around every device
allocation, checked after every run; allocations poisoned with 0xff).  Guards must stay
intact and the results must be bitwise equal -- a kernel reading memory nobody wrote would
see NaN / -1 poison under TQ_GUARD and not under the plain run."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(path, guard):
    env = dict(os.environ, TQ_GUARD="1" if guard else "0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "guard_run.py"), path], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "all ok" in r.stdout


def test_guard_bands_and_poison(tmp_path):
    a, b = str(tmp_path / "plain.npz"), str(tmp_path / "guard.npz")
    run(a, False)
    run(b, True)
    A, B = np.load(a), np.load(b)
    assert set(A.files) == set(B.files)
    for k in A.files:
        assert np.array_equal(A[k], B[k], equal_nan=False), k

"""NEXT-1 (paper-shaped workload and studies) on the GPU: CTR (Alg. 1) through the
engine equals the oracle's gradient descent; the study harness runs end to end and its
outputs have the paper's structure."""
import numpy as np
import pytest

import oracle
from paper_2410_06106_b200 import configs as C
from paper_2410_06106_b200 import studies
from tests.cases import rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec,tol", [(0, 1e-4), (1, 1e-6)])  # tq_get_image returns fp32
def test_ctr_is_alg1_gradient_descent(prec, tol):
    """CTR = one node, no edges: c = 0, b' = 0, so every outer iteration is E1 steps of
    u <- u - eta A^T(A u - d) (Alg. 1) from the previous u -- the oracle's GD."""
    N, n_ang, n_det = 64, 100, 91
    truth, sino = studies.paper_workload(N, n_ang, n_det, 0.0077, 11)
    eta = 1.0 / (2 * n_ang * N)
    r = studies.run_case(truth, sino, n_ang, n_det, 1, e1=10, eta1=eta, iters=3, precision=prec, trace=False)
    u = np.zeros((N, N))
    oracle.build()
    d = sino.astype(np.float64)
    for _ in range(3):
        u = oracle.gd(d, np.zeros((N, N)), 0.0, eta, 10, u, n_ang, np.arange(n_ang))
    assert rel(r["image"], u) <= tol, rel(r["image"], u)


def test_study_harness_structure():
    truth, sino = studies.paper_workload(64, 100, 91, 0.0, 12)
    assert set(np.round(truth.ravel(), 6)) <= set(np.round(np.linspace(0, 1, 257), 6))  # levels + edges
    r2 = studies.run_case(truth, sino, 100, 91, 2, quant=C.Q_KMEANS, k=3, iters=20)
    assert r2["rmse"] < studies.rmse(np.zeros_like(truth), truth)  # it reconstructs
    assert len(r2["rel_change"]) == 20 and r2["rel_change"][-1] < r2["rel_change"][1]
    # K = 3 labels take ceil(log2 3) = 2 bits of 32: 93.75% less than fp32 (plus 12 B of centres)
    assert abs(r2["compression_percent"] - 93.75) < 0.1
    rj = studies.run_case(truth, sino, 100, 91, 2, quant=C.Q_DCT, quality=50, iters=5, jpeg_restart=4)
    assert rj["compression_percent"] > 50.0  # entropy-coded DCT beats the int16 coefficients

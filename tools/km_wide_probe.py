"""The mixed-scale K-means case of tests/test_gpu_kernels.py::test_kmeans_ties_and_extreme_ranges
(same rng stream), plus other seeds: label agreement and centre differences vs the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2410_06106_b200 import tomoq  # noqa: E402


def case(wide, K, tag):
    cen_r, lab_r = oracle.kmeans_encode(wide, K, 10)
    cen, planes, lab = tomoq.kmeans_encode(torch.tensor(wide, device="cuda"), K, 10)
    c = cen.cpu().numpy()
    d = np.abs(c - cen_r.astype(np.float32))
    print(tag, K, "match", np.mean(lab.cpu().numpy() == lab_r), "centres differing", int(np.sum(d > 0)),
          "max |d|", float(d.max()))


rng = np.random.default_rng(3)
rng.integers(0, 3, 5000)
(rng.standard_normal(6000) * 1e-20)
wide = np.concatenate([rng.standard_normal(4000) * 1e6, rng.standard_normal(4000)]).astype(np.float32)
case(wide, 8, "test-stream")
for seed in (3, 4, 5, 6, 7):
    r = np.random.default_rng(seed)
    w = np.concatenate([r.standard_normal(4000) * 1e6, r.standard_normal(4000)]).astype(np.float32)
    for K in (8, 16):
        case(w, K, f"seed{seed}")

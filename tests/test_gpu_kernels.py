"""GPU parity of the single kernels, through the C-ABI, against the fp64 oracle on
identical seeded inputs: projector / backprojector (relative L2 <= 1e-5 in fp32,
north_star), one node's inner solve, and the two codecs (DCT bit-exact, K-means
labels >= 99.99% with dequantized values within 1e-4)."""
import numpy as np
import pytest

import oracle
from paper_2410_06106_b200 import synth, tomoq
from tests.cases import rel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda:0"
TOL = {0: 1e-5, 1: 1e-12}
DT = {0: torch.float32, 1: torch.float64}


def phantom(N, seed, n_e=8, noise=0.05):
    e = synth.random_ellipses(n_e, N, seed)
    img = synth.rasterize(e, N, supersample=2)
    img += noise * np.random.default_rng(seed).standard_normal((N, N))
    return img


def as_input(a, prec):
    """the exact values both sides see: fp32-rounded for the fp32 path"""
    return a.astype(np.float32).astype(np.float64) if prec == 0 else a


PROJ_CASES = [
    (64, 90, 91, None),                       # C1 geometry, all angles
    (64, 90, 91, list(range(0, 23))),         # C1 node 0 (contiguous)
    (40, 33, 57, [0, 5, 8, 16, 17, 24, 32]),  # ragged tile tails, odd angle count
    (37, 20, 53, None),                       # N not a multiple of 8 (stateless API allows it)
    (256, 180, 363, list(range(3, 180, 8))),  # C2 node 3 (round-robin)
    (8, 4, 13, None),                         # tiny, includes the 45 degree tie
    (64, 180, 91, None),                      # > 64 angles per orientation: several forward and backward batches
    (200, 100, 283, None),                    # N not a multiple of the 128 x 32 / 64 x 64 tiles (TMA zero fill)
]


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("N,n_ang,n_det,sel", PROJ_CASES)
def test_project_backproject_parity(N, n_ang, n_det, sel, prec):
    img = as_input(phantom(N, N + n_ang), prec)
    sel_a = np.arange(n_ang) if sel is None else np.asarray(sel)
    ref = oracle.project(img, n_ang, n_det, sel_a)
    got = tomoq.project(torch.tensor(img, dtype=DT[prec], device=DEV), n_ang, n_det, sel_a)
    assert rel(got.cpu().numpy(), ref) <= TOL[prec]
    y = as_input(np.random.default_rng(N).standard_normal((len(sel_a), n_det)), prec)
    refb = oracle.backproject(y, N, n_ang, sel_a)
    gotb = tomoq.backproject(torch.tensor(y, dtype=DT[prec], device=DEV), N, n_ang, sel_a)
    assert rel(gotb.cpu().numpy(), refb) <= TOL[prec]


@pytest.mark.parametrize("prec", [0, 1])
def test_project_unaligned_input(prec):
    """A caller's image that is not 16-byte aligned takes the scalar staging path."""
    N, n_ang, n_det = 64, 30, 91
    img = as_input(phantom(N, 77), prec)
    buf = torch.zeros(N * N + 1, dtype=DT[prec], device=DEV)
    buf[1:] = torch.tensor(img.ravel(), dtype=DT[prec], device=DEV)
    view = buf[1:].view(N, N)
    assert view.data_ptr() % 16 != 0
    got = tomoq.project(view, n_ang, n_det)
    assert rel(got.cpu().numpy(), oracle.project(img, n_ang, n_det)) <= TOL[prec]


def test_adjoint_identity_fp32_and_fp64():
    N, n_ang, n_det = 128, 60, 183
    rng = np.random.default_rng(9)
    for prec, tol in ((0, 1e-5), (1, 1e-12)):
        x = torch.tensor(rng.standard_normal((N, N)), dtype=DT[prec], device=DEV)
        y = torch.tensor(rng.standard_normal((n_ang, n_det)), dtype=DT[prec], device=DEV)
        lhs = float((tomoq.project(x, n_ang, n_det) * y).double().sum())
        rhs = float((x * tomoq.backproject(y, N, n_ang)).double().sum())
        assert abs(lhs - rhs) <= tol * abs(lhs)


@pytest.mark.parametrize("N,n_ang,n_det,sel", [
    (1024, 90, 1449, [0, 8, 40, 88]),           # C4 (G=1) node 0 sample of its angles
    (2048, 1500, 2897, [0, 376, 752, 1128]),    # C5 node 0 sample
])
def test_projector_full_size_sampled(N, n_ang, n_det, sel):
    """BASELINE sizes: the oracle computes a sample of the angles in full."""
    img = as_input(phantom(N, 5, n_e=30), 0)
    ref = oracle.project(img, n_ang, n_det, sel)
    timg = torch.tensor(img, dtype=torch.float32, device=DEV)
    got = tomoq.project(timg, n_ang, n_det, sel)
    assert rel(got.cpu().numpy(), ref) <= 1e-5
    y = as_input(ref / ref.max(), 0)
    refb = oracle.backproject(y, N, n_ang, sel)
    gotb = tomoq.backproject(torch.tensor(y, dtype=torch.float32, device=DEV), N, n_ang, sel)
    assert rel(gotb.cpu().numpy(), refb) <= 1e-5


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("inner,e1", [(tomoq.INNER_CG, 5), (tomoq.INNER_GD, 10), (tomoq.INNER_CG, 0),
                                     (tomoq.INNER_CG, 1), (tomoq.INNER_CG, 2)])
def test_local_solve_parity(prec, inner, e1):
    N, n_ang, n_det = 128, 90, 183
    sel = list(range(2, 90, 8))
    rng = np.random.default_rng(4)
    truth = phantom(N, 11)
    d = as_input(oracle.project(truth, n_ang, n_det, sel) + 0.1 * rng.standard_normal((len(sel), n_det)), prec)
    bp = as_input(rng.standard_normal(N * N) * 0.5, prec)
    x0 = as_input(truth + 0.1 * rng.standard_normal((N, N)), prec)
    c, eta = 2.0, 1.0 / (2 * len(sel) * N + 2.0)
    if inner == tomoq.INNER_CG:
        ref = oracle.cg(d, bp, c, e1, x0, n_ang, sel)
    else:
        ref = oracle.gd(d, bp, c, eta, e1, x0, n_ang, sel)
    T = lambda a: torch.tensor(a, dtype=DT[prec], device=DEV)
    got = tomoq.local_solve(T(d), T(bp.reshape(N, N)), c, e1, T(x0), n_ang, sel, inner=inner, eta=eta)
    assert rel(got.cpu().numpy(), ref) <= (1e-5 if prec == 0 else 1e-11)


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("inner,e1", [(tomoq.INNER_CG, 3), (tomoq.INNER_GD, 4)])
def test_local_solve_many_angles(prec, inner, e1):
    """45 angles on one node: the backprojector's angle batches (32 per batch for the CG
    epilogue, 16 for the residual / GD epilogues in fp32) span several staging rounds."""
    N, n_ang, n_det = 96, 90, 137
    sel = list(range(1, 90, 2))
    rng = np.random.default_rng(7)
    truth = phantom(N, 5)
    d = as_input(oracle.project(truth, n_ang, n_det, sel) + 0.1 * rng.standard_normal((len(sel), n_det)), prec)
    bp = as_input(rng.standard_normal(N * N) * 0.5, prec)
    x0 = as_input(truth + 0.1 * rng.standard_normal((N, N)), prec)
    c, eta = 1.5, 1.0 / (2 * len(sel) * N + 1.5)
    if inner == tomoq.INNER_CG:
        ref = oracle.cg(d, bp, c, e1, x0, n_ang, sel)
    else:
        ref = oracle.gd(d, bp, c, eta, e1, x0, n_ang, sel)
    T = lambda a: torch.tensor(a, dtype=DT[prec], device=DEV)
    got = tomoq.local_solve(T(d), T(bp.reshape(N, N)), c, e1, T(x0), n_ang, sel, inner=inner, eta=eta)
    assert rel(got.cpu().numpy(), ref) <= (1e-5 if prec == 0 else 1e-11)


# ---------------------------------------------------------------- codecs
def kmeans_input(n, seed):
    rng = np.random.default_rng(seed)
    N = int(np.ceil(np.sqrt(n)))
    img = phantom(max(N, 8), seed, noise=0.02).ravel()[:n]
    return (img + 1e-3 * rng.standard_normal(n)).astype(np.float32)


@pytest.mark.parametrize("n,K,iters", [(5, 2, 10), (1000, 1, 3), (1000, 16, 10), (65536, 16, 10),
                                       (65537, 64, 10), (4099, 3, 0), (1 << 20, 64, 10),
                                       (20000, 100, 5), (3000, 256, 4),
                                       (2048 * 2048, 32, 10)])  # config 5 payload (a 2048^2 slice)
def test_kmeans_parity(n, K, iters):
    v = kmeans_input(n, n + K)
    cen_r, lab_r = oracle.kmeans_encode(v, K, iters)
    cen, planes, lab = tomoq.kmeans_encode(torch.tensor(v, device=DEV), K, iters)
    lab = lab.cpu().numpy()
    assert np.mean(lab == lab_r) >= 0.9999
    assert np.max(np.abs(cen.cpu().numpy() - cen_r)) <= 1e-4 * max(1.0, np.abs(v).max())
    dec = tomoq.kmeans_decode(cen, planes, n, K).cpu().numpy()
    assert np.array_equal(dec, cen.cpu().numpy()[lab])  # bit-planes carry exactly the labels
    assert np.max(np.abs(dec - oracle.kmeans_decode(cen_r, lab_r))[lab == lab_r]) <= 1e-4


def test_kmeans_spec_example_and_edges():
    cen, planes, lab = tomoq.kmeans_encode(torch.tensor([0, 0, 1, 1, 10], dtype=torch.float32, device=DEV), 2, 10)
    assert sorted(cen.cpu().tolist()) == [0.5, 10.0]
    assert tomoq.kmeans_decode(cen, planes, 5, 2).cpu().tolist() == [0.5, 0.5, 0.5, 0.5, 10.0]
    const = torch.full((777,), 2.5, device=DEV)
    cen, planes, lab = tomoq.kmeans_encode(const, 8, 10)
    assert np.all(tomoq.kmeans_decode(cen, planes, 777, 8).cpu().numpy() == 2.5)
    neg = torch.tensor(-np.abs(kmeans_input(3333, 1)) - 5, device=DEV)
    cr, lr = oracle.kmeans_encode(neg.cpu().numpy(), 7, 6)
    c, p, l = tomoq.kmeans_encode(neg, 7, 6)
    assert np.mean(l.cpu().numpy() == lr) >= 0.9999


@pytest.mark.parametrize("rows,cols,q", [(2048, 2048, 75), (1024, 1024, 50)])  # configs 5 and 4 sizes
def test_dct_bit_exact_full_size(rows, cols, q):
    test_dct_bit_exact(rows, cols, q)


@pytest.mark.parametrize("rows,cols", [(8, 8), (64, 64), (16, 512), (512, 512), (256, 64)])
@pytest.mark.parametrize("q", [1, 25, 50, 75, 100])
def test_dct_bit_exact(rows, cols, q):
    v = (phantom(max(rows, cols), rows + q, noise=0.03)[:rows, :cols] * 3 - 1).astype(np.float32)
    coef_r, mm_r = oracle.dct_encode(v, q)
    coef, mm = tomoq.dct_encode(torch.tensor(v, device=DEV), q)
    assert np.array_equal(mm.cpu().numpy(), mm_r)
    assert np.array_equal(coef.cpu().numpy(), coef_r)
    dec_r = oracle.dct_decode(coef_r, mm_r, rows, cols, q)
    dec = tomoq.dct_decode(coef, mm, rows, cols, q).cpu().numpy()
    assert np.array_equal(dec, dec_r)


def test_dct_constant_and_extremes():
    v = np.full((16, 16), -3.5, np.float32)
    coef, mm = tomoq.dct_encode(torch.tensor(v, device=DEV), 50)
    assert not torch.any(coef) and np.all(tomoq.dct_decode(coef, mm, 16, 16, 50).cpu().numpy() == -3.5)
    v = np.zeros((8, 16), np.float32)
    v[0, 0], v[7, 15] = -1e30, 1e30
    coef_r, mm_r = oracle.dct_encode(v, 75)
    coef, mm = tomoq.dct_encode(torch.tensor(v, device=DEV), 75)
    assert np.array_equal(coef.cpu().numpy(), coef_r)


# ----------------------------------------------------------------- JPEG entropy coding (NEXT-2)
@pytest.mark.parametrize("rows,cols,q", [(64, 64, 50), (512, 512, 50), (256, 512, 75), (2048, 2048, 75),
                                         (8, 8, 100), (40, 24, 10)])
@pytest.mark.parametrize("restart", [1, 4, 16])
def test_jpeg_entropy_bit_exact(rows, cols, q, restart):
    """GPU entropy-coded segment == the oracle's byte for byte (coefficients of the DCT
    quantizer on the phantom recipe, several sizes, qualities and restart intervals);
    the GPU decoder returns the coefficients of both streams."""
    v = (phantom(max(rows, cols), rows + q, noise=0.03)[:rows, :cols] * 3 - 1).astype(np.float32)
    coef_r, _ = oracle.dct_encode(v, q)
    nb = rows * cols // 64
    ref = oracle.jpeg_encode(coef_r, restart)
    got = tomoq.jpeg_encode(torch.tensor(coef_r, device=DEV), restart).cpu().numpy().tobytes()
    assert got == ref
    dec = tomoq.jpeg_decode(torch.tensor(np.frombuffer(ref, np.uint8).copy(), device=DEV), nb, restart)
    assert np.array_equal(dec.cpu().numpy(), coef_r)


@pytest.mark.parametrize("restart", [1, 3, 64, 128, 129, 200])
def test_jpeg_entropy_dense_blocks_and_stuffing(restart):
    """Dense blocks (every AC coefficient non-zero, categories 1..7 -- up to ~950 coded
    bits per block, so long intervals cycle the warp coder's bit ring many times) mixed
    with sparse and all-zero blocks and values chosen so 0xFF bytes (stuffed 0x00) are
    frequent; byte-identical to the oracle's sequential coder, decoded back exactly."""
    rng = np.random.default_rng(restart)
    nb = 300
    c = np.zeros((nb, 64), np.int16)
    kind = rng.integers(0, 4, size=nb)
    for b in range(nb):
        if kind[b] == 0:    # dense, random categories
            mag = rng.integers(1, 128, size=64)
            c[b] = mag * rng.choice([-1, 1], size=64)
        elif kind[b] == 1:  # all ones: long runs of 1-bits (0xFF bytes) in the codes
            c[b] = -1
        elif kind[b] == 2:  # sparse with long zero runs (ZRL)
            idx = rng.choice(64, size=3, replace=False)
            c[b, idx] = rng.integers(-300, 300, size=3)
    c[:, 0] = rng.integers(-1000, 1000, size=nb)
    flat = c.ravel()
    ref = oracle.jpeg_encode(flat, restart)
    assert ref.count(b"\xff\x00") > 10
    got = tomoq.jpeg_encode(torch.tensor(flat, device=DEV), restart).cpu().numpy().tobytes()
    assert got == ref
    back = tomoq.jpeg_decode(torch.tensor(np.frombuffer(ref, np.uint8).copy(), device=DEV), nb, restart)
    assert np.array_equal(back.cpu().numpy(), flat)


def test_jpeg_entropy_extremes_and_errors():
    zz = oracle.jpeg_zigzag()
    rng = np.random.default_rng(7)
    c = np.zeros((33, 64), np.int16)
    c[:, 0] = rng.integers(-1024, 1017, size=33)          # DC differences up to 11 bits
    c[0, zz[1]], c[1, zz[17]], c[2, zz[63]] = 1023, -1023, 7  # AC category 10, no EOB
    c[3, zz[16]], c[3, zz[33]], c[4, zz[62]] = 1, -2, 3     # ZRL runs
    c[5:] *= 1
    flat = c.ravel()
    for r in (1, 2, 7, 64):
        ref = oracle.jpeg_encode(flat, r)
        got = tomoq.jpeg_encode(torch.tensor(flat, device=DEV), r).cpu().numpy().tobytes()
        assert got == ref
        back = tomoq.jpeg_decode(torch.tensor(np.frombuffer(ref, np.uint8).copy(), device=DEV), 33, r)
        assert np.array_equal(back.cpu().numpy(), flat)
    bad = np.zeros(64, np.int16)
    bad[1] = 1024
    with pytest.raises(tomoq.TomoQError):
        tomoq.jpeg_encode(torch.tensor(bad, device=DEV), 1)
    s = oracle.jpeg_encode(flat, 4)
    broken = np.frombuffer(s, np.uint8).copy()
    k = bytes(broken).index(b"\xff\xd1")
    broken[k + 1] = 0xD3  # misnumbered RSTm
    with pytest.raises(tomoq.TomoQError):
        tomoq.jpeg_decode(torch.tensor(broken, device=DEV), 33, 4)


# ----------------------------------------------------------------- Siddon (NEXT-3, R-26)
SIDDON_CASES = [
    (64, 90, 91, None),                       # C1 geometry: theta = 0 / pi/2 rays on pixel edges
    (64, 90, 92, list(range(0, 90, 4))),      # even n_det: axis rays through pixel centres
    (40, 33, 57, [0, 5, 8, 16, 17, 24, 32]),  # ragged tiles
    (37, 20, 53, None),                       # odd N
    (8, 4, 13, None),                         # 45 degree rays through corners
    (256, 180, 363, list(range(3, 180, 8))),  # C2 node 3
    (200, 100, 283, None),
]


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("N,n_ang,n_det,sel", SIDDON_CASES)
def test_siddon_project_backproject_parity(N, n_ang, n_det, sel, prec):
    img = as_input(phantom(N, N + n_ang + 1), prec)
    sel_a = np.arange(n_ang) if sel is None else np.asarray(sel)
    ref = oracle.project_siddon(img, n_ang, n_det, sel_a)
    got = tomoq.project(torch.tensor(img, dtype=DT[prec], device=DEV), n_ang, n_det, sel_a,
                        projector=tomoq.PROJ_SIDDON)
    assert rel(got.cpu().numpy(), ref) <= TOL[prec]
    y = as_input(np.random.default_rng(N + 1).standard_normal((len(sel_a), n_det)), prec)
    refb = oracle.backproject_siddon(y, N, n_ang, sel_a)
    gotb = tomoq.backproject(torch.tensor(y, dtype=DT[prec], device=DEV), N, n_ang, sel_a,
                             projector=tomoq.PROJ_SIDDON)
    assert rel(gotb.cpu().numpy(), refb) <= TOL[prec]


def test_siddon_axis_rays_exact_half_split():
    """theta = 0 and pi/2 with even N, odd n_det: every ray on a pixel edge takes half of
    each neighbouring column / row (R-26) -- exactly, in fp32 and fp64."""
    N, n_ang, n_det = 32, 8, 47
    img = phantom(N, 5)
    for prec in (0, 1):
        x = as_input(img, prec)
        got = tomoq.project(torch.tensor(x, dtype=DT[prec], device=DEV), n_ang, n_det, [0, 4],
                            projector=tomoq.PROJ_SIDDON).cpu().numpy()
        ref = oracle.project_siddon(x, n_ang, n_det, [0, 4])
        assert np.max(np.abs(got - ref)) <= (2e-5 if prec == 0 else 1e-12) * np.abs(ref).max()


@pytest.mark.parametrize("n,K", [(1 << 20, 64), (2048 * 2048, 32)])
def test_kmeans_encode_bitwise_repeatable(n, K):
    """The first radix pass ranks keys with shared-memory atomics, so the order of equal keys
    inside a sort group differs from call to call; every output (centres, bit-planes, labels)
    must not: repeated encodes of the same payload are bitwise equal (R-16)."""
    v = torch.tensor(kmeans_input(n, 11 + K), device=DEV)
    outs = [tomoq.kmeans_encode(v, K, 10) for _ in range(3)]
    for cen, planes, lab in outs[1:]:
        assert torch.equal(cen, outs[0][0]) and torch.equal(planes, outs[0][1]) and torch.equal(lab, outs[0][2])


def test_kmeans_ties_and_extreme_ranges():
    """Values equal to a threshold go to the lower cluster on both sides (R-16); the final
    assignment's bucket map stays exact when the payload range overflows fp32 (max - min =
    inf) or is a handful of discrete levels.  (Cluster sums are fixed-point integers with
    resolution 2^(E + ceil(log2 n) - 62), E = exponent of max|v| -- DESIGN.md R-16.  Values
    1e6 times smaller than the largest keep ~27 fractional bits: their rounding moves a
    cluster sum far below the fp32 resolution of its centre, so 1e6-scale mixed with O(1)
    values is held to the north_star's label bar (measured: identical centres and labels,
    tools/km_wide_probe.py); a payload mixing +-3e38 with O(1) values loses the O(1) values
    entirely, so that case checks only the assignment against the GPU's own centres.)"""
    rng = np.random.default_rng(3)
    for v, K in ((rng.integers(0, 3, 5000).astype(np.float32), 2),           # {0, 1, 2}: thresholds hit values
                 (np.repeat(np.arange(10, dtype=np.float32), 300), 4),       # ten levels
                 ((rng.standard_normal(6000) * 1e-20).astype(np.float32), 16)):  # tiny values
        cen_r, lab_r = oracle.kmeans_encode(v, K, 10)
        cen, planes, lab = tomoq.kmeans_encode(torch.tensor(v, device=DEV), K, 10)
        assert np.array_equal(lab.cpu().numpy(), lab_r)
        assert np.array_equal(cen.cpu().numpy(), cen_r.astype(np.float32))
    wide = np.concatenate([rng.standard_normal(4000) * 1e6, rng.standard_normal(4000)]).astype(np.float32)
    cases = [(wide, 8)]
    for seed in (4, 5, 6):
        r = np.random.default_rng(seed)
        cases.append((np.concatenate([r.standard_normal(4000) * 1e6, r.standard_normal(4000)]).astype(np.float32), 16))
    for w, K in cases:
        cen_r, lab_r = oracle.kmeans_encode(w, K, 10)
        cen, planes, lab = tomoq.kmeans_encode(torch.tensor(w, device=DEV), K, 10)
        assert np.mean(lab.cpu().numpy() == lab_r) >= 0.9999
        assert np.max(np.abs(cen.cpu().numpy() - cen_r) / np.maximum(np.abs(cen_r), 1.0)) <= 1e-6
    huge = np.concatenate([rng.standard_normal(4000), [3.0e38, -3.0e38]]).astype(np.float32)
    cen, planes, lab = tomoq.kmeans_encode(torch.tensor(huge, device=DEV), 8, 10)
    c = cen.cpu().numpy().astype(np.float64)
    thr = np.sort(((c[:-1] + c[1:]) * 0.5).astype(np.float32))
    want = np.searchsorted(thr, huge, side="left")  # label = #{k : v > thr_k}
    assert np.array_equal(lab.cpu().numpy(), want)

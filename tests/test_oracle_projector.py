"""Pins of the oracle's projector A (Joseph, ray-driven) and backprojector A^T
(pixel-driven closed form) against things other than themselves: a brute-force
dense matrix built from the geometric definition, the continuous x-ray transform
(Eq. 1) of disks / ellipses / Gaussians in closed form, exact special
cases, and the adjoint identity that ties the two independent algorithms."""
import math

import numpy as np
import pytest

import oracle
from paper_2410_06106_b200 import synth


def dense_joseph(N, n_ang, n_det):
    """Brute force: for every ray and pixel, Joseph's interpolation weight from the
    geometry -- walk the ray's major-axis lines and give the pixel its linear
    interpolation weight times the per-line ray length (independent of oracle.c)."""
    A = np.zeros((n_ang * n_det, N * N))
    half = (N - 1) / 2.0
    for a in range(n_ang):
        th = math.pi * a / n_ang
        c, s = math.cos(th), math.sin(th)
        xmaj = 4 * a >= n_ang and 4 * a <= 3 * n_ang
        for j in range(n_det):
            t = j - (n_det - 1) / 2.0
            if not xmaj:
                for r in range(N):
                    y = half - r
                    x = (t - y * s) / c           # where the ray meets row r
                    col = x + half
                    for cc in range(N):
                        w = max(0.0, 1.0 - abs(col - cc))
                        A[a * n_det + j, r * N + cc] += w / abs(c)
            else:
                for cc in range(N):
                    x = cc - half
                    y = (t - x * c) / s
                    row = half - y
                    for r in range(N):
                        w = max(0.0, 1.0 - abs(row - r))
                        A[a * n_det + j, r * N + cc] += w / abs(s)
    return A


@pytest.mark.parametrize("N,n_ang,n_det", [(8, 8, 13), (8, 12, 12), (10, 7, 15)])
def test_project_equals_bruteforce_dense(N, n_ang, n_det):
    A = dense_joseph(N, n_ang, n_det)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((N, N))
    y = rng.standard_normal((n_ang, n_det))
    np.testing.assert_allclose(oracle.project(x, n_ang, n_det).ravel(), A @ x.ravel(),
                               rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.backproject(y, N, n_ang).ravel(), A.T @ y.ravel(),
                               rtol=0, atol=1e-12)


def test_closed_form_support_at_most_two_bins():
    """Each (pixel, angle) touches <= 2 bins and the weights of one pixel's column sum
    to at most 1/m (bounded by sqrt 2)."""
    N, n_ang, n_det = 12, 16, 17
    A = dense_joseph(N, n_ang, n_det).reshape(n_ang, n_det, N * N)
    nnz = (A > 0).sum(axis=1)
    assert nnz.max() <= 2
    _, _, _, _, m = oracle.angles(n_ang)
    assert np.all(A.sum(axis=1) <= (1.0 / m)[:, None] + 1e-12)


@pytest.mark.parametrize("N,n_ang,n_det", [(16, 24, 23), (33, 17, 47), (64, 90, 91)])
def test_adjoint_identity_fp64(N, n_ang, n_det):
    rng = np.random.default_rng(N)
    sel = np.sort(rng.choice(n_ang, size=max(1, n_ang // 3), replace=False))
    for _ in range(5):
        x = rng.standard_normal((N, N))
        y = rng.standard_normal((len(sel), n_det))
        lhs = np.vdot(oracle.project(x, n_ang, n_det, sel), y)
        rhs = np.vdot(x, oracle.backproject(y, N, n_ang, sel))
        assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), 1e-300) + 1e-12


def test_constant_image_central_ray():
    """Constant image u = 1: the central ray (t = 0) crosses all N major-axis lines
    fully inside the grid, so its Joseph integral is exactly N / m_a."""
    N, n_ang, n_det = 64, 36, 91
    s = oracle.project(np.ones((N, N)), n_ang, n_det)
    _, _, _, _, m = oracle.angles(n_ang)
    np.testing.assert_allclose(s[:, n_det // 2], N / m, rtol=1e-13)


def test_affine_image_central_ray():
    """u = a + b x + c y is odd-symmetric about the centre except for a; the
    central ray's integral is a N / m_a (the linear terms cancel in the sum)."""
    N, n_ang, n_det = 64, 36, 91
    xs, ys = synth.pixel_centres(N)
    img = 0.7 + 0.3 * xs[None, :] - 0.2 * ys[:, None]
    s = oracle.project(img, n_ang, n_det)
    _, _, _, _, m = oracle.angles(n_ang)
    np.testing.assert_allclose(s[:, n_det // 2], 0.7 * N / m, rtol=1e-12)


def test_theta_zero_is_interpolated_column_sums():
    """theta = 0: rays are the vertical lines x = t, so d_j is the linear
    interpolation of the column-sum profile at x = t_j."""
    N, n_det = 32, 47
    rng = np.random.default_rng(1)
    img = rng.random((N, N))
    s = oracle.project(img, 4, n_det, sel=[0])[0]
    xs, _ = synth.pixel_centres(N)
    colsum = img.sum(axis=0)
    t = synth.bin_centres(n_det)
    expect = np.interp(t, xs, colsum, left=0.0, right=0.0)
    # outside [x_0 - 1, x_{N-1} + 1] the profile is 0; within one pixel of the edge it
    # ramps linearly to 0 (a tap falls off the grid)
    edge = np.interp(t, np.r_[xs[0] - 1, xs, xs[-1] + 1], np.r_[0, colsum, 0])
    np.testing.assert_allclose(s, edge, atol=1e-12)
    inner = (t >= xs[0]) & (t <= xs[-1])
    np.testing.assert_allclose(s[inner], expect[inner], atol=1e-12)


@pytest.mark.parametrize("shape", ["disk", "ellipse"])
def test_analytic_chord_lengths(shape):
    """North_star pin: 4x4-supersampled raster of a disk / rotated ellipse, projected
    by the oracle, vs the closed-form line integral rho 2ab sqrt(s^2 - tau^2)/s^2.
    Bound: RMSE <= 0.5% of the peak over all angles (SPEC.md:73 allows 2%)."""
    N, n_ang = 256, 180
    n_det = 363
    if shape == "disk":
        e = synth.Ellipses(np.array([10.3]), np.array([-7.9]), np.array([60.0]),
                           np.array([60.0]), np.array([0.0]), np.array([1.0]))
    else:
        e = synth.Ellipses(np.array([-12.5]), np.array([20.25]), np.array([70.0]),
                           np.array([35.0]), np.array([0.6]), np.array([0.8]))
    img = synth.rasterize(e, N)
    th = synth.default_angles(n_ang)
    ref = synth.ellipse_sinogram(e, th, n_det)
    got = oracle.project(img, n_ang, n_det)
    rmse = np.sqrt(np.mean((got - ref) ** 2))
    assert rmse <= 0.005 * ref.max(), rmse / ref.max()
    # the worst rays are the near-tangent ones, where the chord ~ sqrt(s - |tau|) is not
    # resolved by a pixel raster; bound the max error loosely
    assert np.max(np.abs(got - ref)) <= 0.08 * ref.max()


def test_gaussian_blob():
    """Gaussian exp(-r^2/2 sigma^2), sigma = 20 px, sampled at pixel centres: the
    continuous transform is sqrt(2 pi) sigma exp(-t^2 / 2 sigma^2) at every angle."""
    N, n_ang, n_det, sig = 256, 30, 363, 20.0
    xs, ys = synth.pixel_centres(N)
    img = np.exp(-(xs[None, :] ** 2 + ys[:, None] ** 2) / (2 * sig * sig))
    got = oracle.project(img, n_ang, n_det)
    t = synth.bin_centres(n_det)
    ref = math.sqrt(2 * math.pi) * sig * np.exp(-t * t / (2 * sig * sig))
    assert np.max(np.abs(got - ref[None, :])) <= 5e-4 * ref.max()


def test_linearity_nonnegativity():
    N, n_ang, n_det = 24, 20, 35
    rng = np.random.default_rng(3)
    u, w = rng.random((N, N)), rng.random((N, N))
    Au, Aw = oracle.project(u, n_ang, n_det), oracle.project(w, n_ang, n_det)
    np.testing.assert_allclose(oracle.project(2.5 * u - 1.5 * w, n_ang, n_det), 2.5 * Au - 1.5 * Aw,
                               atol=1e-12)
    assert Au.min() >= 0.0
    assert oracle.backproject(np.abs(Au), N, n_ang).min() >= 0.0


def test_zero_inputs():
    assert not np.any(oracle.project(np.zeros((16, 16)), 8, 23))
    assert not np.any(oracle.backproject(np.zeros((8, 23)), 16, 8))


# ----------------------------------------------------------------- Siddon (NEXT-3, R-26)
from tests.helpers import clip_length, dense_siddon  # noqa: E402


@pytest.mark.parametrize("N,n_ang,n_det", [(6, 8, 9), (8, 12, 12), (7, 10, 11), (8, 4, 13)])
def test_siddon_equals_bruteforce_clipping(N, n_ang, n_det):
    """P_ji = length of ray j inside pixel i: the oracle's Siddon crossing
    lists vs clipping each ray against each pixel square; odd and even N and n_det put
    rays on pixel edges (theta = 0, pi/2), through corners (pi/4) and in general position."""
    A = dense_siddon(N, n_ang, n_det)
    rng = np.random.default_rng(N * 100 + n_ang)
    img = rng.random((N, N))
    got = oracle.project_siddon(img, n_ang, n_det)
    np.testing.assert_allclose(got.ravel(), A @ img.ravel(), rtol=0, atol=1e-12)
    sino = rng.random((n_ang, n_det))
    np.testing.assert_allclose(oracle.backproject_siddon(sino, N, n_ang).ravel(), A.T @ sino.ravel(),
                               rtol=0, atol=1e-12)


def test_siddon_chord_sums():
    """Sum over pixels of P_ji = length of ray j inside the image square,
    for 2000 random rays: the projection of the all-ones image."""
    N, n_ang, n_det = 32, 250, 47
    ones = np.ones((N, N))
    got = oracle.project_siddon(ones, n_ang, n_det)
    h = N / 2
    for a in range(n_ang):
        cs, sn = (1.0, 0.0) if a == 0 else ((0.0, 1.0) if 2 * a == n_ang else
                                            (math.cos(math.pi * a / n_ang), math.sin(math.pi * a / n_ang)))
        for j in range(0, n_det, 6):
            t = j - 0.5 * (n_det - 1)
            want = clip_length(-h, h, -h, h, t * cs, t * sn, -sn, cs)
            # a ray on the outer boundary line keeps half (its outer neighbour is absent)
            if (sn == 0 and abs(t * cs) == h) or (cs == 0 and abs(t * sn) == h):
                want *= 0.5
            assert abs(got[a, j] - want) <= 1e-12 * max(1.0, want), (a, j)


def test_siddon_axis_rays_are_half_column_sums():
    """theta = 0 with even N and odd n_det: every ray lies on a column boundary, so its
    value is the mean of the two adjacent column sums (R-26)."""
    N, n_ang, n_det = 16, 6, 23
    img = np.random.default_rng(3).random((N, N))
    s = oracle.project_siddon(img, n_ang, n_det)
    cols = np.concatenate([[0.0], img.sum(axis=0), [0.0]])
    for j in range(n_det):
        t = j - (n_det - 1) // 2
        k = int(t + N // 2)  # boundary index 0..N
        want = 0.5 * (cols[k] + cols[k + 1]) if 0 <= k <= N else 0.0
        assert abs(s[0, j] - want) <= 1e-12
    rows = np.concatenate([[0.0], img.sum(axis=1)[::-1], [0.0]])  # bottom row first (y up)
    for j in range(n_det):  # theta = pi/2: rays y = t on row boundaries
        t = j - (n_det - 1) // 2
        k = int(t + N // 2)
        want = 0.5 * (rows[k] + rows[k + 1]) if 0 <= k <= N else 0.0
        assert abs(s[3, j] - want) <= 1e-12


@pytest.mark.parametrize("shape", ["disk", "ellipse"])
def test_siddon_analytic_chord_lengths(shape):
    """As for Joseph: a supersampled disk / rotated ellipse vs the closed-form line
    integral (RMSE <= 0.5% of the peak)."""
    N, n_ang, n_det = 256, 180, 363
    if shape == "disk":
        e = synth.Ellipses(np.array([10.3]), np.array([-7.9]), np.array([60.0]),
                           np.array([60.0]), np.array([0.0]), np.array([1.0]))
    else:
        e = synth.Ellipses(np.array([-12.5]), np.array([20.25]), np.array([70.0]),
                           np.array([35.0]), np.array([0.6]), np.array([0.8]))
    img = synth.rasterize(e, N)
    ref = synth.ellipse_sinogram(e, synth.default_angles(n_ang), n_det)
    got = oracle.project_siddon(img, n_ang, n_det)
    assert np.sqrt(np.mean((got - ref) ** 2)) <= 0.005 * ref.max()


def test_siddon_adjoint_and_admm_runs():
    N, n_ang, n_det = 24, 30, 35
    rng = np.random.default_rng(9)
    x, y = rng.random((N, N)), rng.random((n_ang, n_det))
    lhs = np.sum(oracle.project_siddon(x, n_ang, n_det) * y)
    rhs = np.sum(x * oracle.backproject_siddon(y, N, n_ang))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    # the ADMM loop with the Siddon projector: graph rule converges towards the Siddon
    # least-squares solution on a tiny problem
    N, n_ang, n_det = 8, 16, 13
    A = dense_siddon(N, n_ang, n_det)
    xt = rng.random(N * N)
    sino = (A @ xt).reshape(n_ang, n_det)
    edges = [(0, 1), (1, 2), (2, 3), (3, 0)]
    o = oracle.OracleADMM(N, n_det, n_ang, 4, edges, sino, False, rule=0, inner=1, e1=5, rho=0.1,
                          projector=1).run(3000)
    ls = np.linalg.lstsq(A, sino.ravel(), rcond=None)[0]
    assert np.linalg.norm(o.image().ravel() - ls) <= 1e-4 * np.linalg.norm(ls)


# ---------------------------------------------------------------- explicit angle lists
def explicit_angles(n, seed):
    """Seeded irregular angles in [0, pi) including the special ones (0, pi/4, pi/2, 3pi/4)."""
    rng = np.random.default_rng(seed)
    t = np.concatenate([[0.0, math.pi / 4, math.pi / 2, 3 * math.pi / 4], rng.uniform(0, math.pi, n - 4)])
    return t


@pytest.mark.parametrize("N,n_det,seed", [(8, 13, 1), (9, 15, 2)])
def test_explicit_angles_equal_bruteforce_dense(N, n_det, seed):
    """tq_geometry.angles_rad / the oracle's theta list: the brute-force Joseph matrix built
    from the same explicit angles (major axis |sin| >= |cos|, R-3), forward and transpose."""
    from tests.helpers import dense_joseph
    theta = explicit_angles(10, seed)
    A = dense_joseph(N, len(theta), n_det, theta=theta)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((N, N))
    y = rng.standard_normal((len(theta), n_det))
    np.testing.assert_allclose(oracle.project(x, len(theta), n_det, theta=theta).ravel(), A @ x.ravel(),
                               rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.backproject(y, N, len(theta), theta=theta).ravel(), A.T @ y.ravel(),
                               rtol=0, atol=1e-12)


def test_explicit_uniform_list_equals_uniform_angles():
    """An explicit list equal to pi a / n (no angle on the 45-degree tie) gives the uniform run."""
    N, n_ang, n_det = 32, 90, 47
    x = np.random.default_rng(3).standard_normal((N, N))
    theta = math.pi * np.arange(n_ang) / n_ang
    np.testing.assert_array_equal(oracle.project(x, n_ang, n_det, theta=theta), oracle.project(x, n_ang, n_det))


def test_explicit_angles_analytic_ellipse():
    """Irregular angles: a 4x4-supersampled rotated ellipse vs its closed-form line integrals
    (Eq. 1) at those angles, with the bound of test_analytic_chord_lengths."""
    N, n_det = 256, 363
    e = synth.Ellipses(np.array([-12.5]), np.array([20.25]), np.array([70.0]),
                       np.array([35.0]), np.array([0.6]), np.array([0.8]))
    img = synth.rasterize(e, N)
    theta = explicit_angles(24, 7)
    ref = synth.ellipse_sinogram(e, theta, n_det)
    got = oracle.project(img, len(theta), n_det, theta=theta)
    assert np.sqrt(np.mean((got - ref) ** 2)) <= 0.005 * ref.max()
    assert np.max(np.abs(got - ref)) <= 0.08 * ref.max()


def test_explicit_angles_adjoint_and_siddon_dense():
    """Explicit angles: the fp64 adjoint identity (north_star, 1e-10) and Siddon's matrix
    against the per-pixel clip of every ray (axis rays on pixel edges half-split)."""
    from tests.helpers import dense_siddon
    theta = explicit_angles(8, 5)
    N, n_det = 8, 13
    rng = np.random.default_rng(11)
    x = rng.standard_normal((N, N))
    y = rng.standard_normal((len(theta), n_det))
    lhs = float(np.sum(oracle.project(x, len(theta), n_det, theta=theta) * y))
    rhs = float(np.sum(x * oracle.backproject(y, N, len(theta), theta=theta)))
    assert abs(lhs - rhs) <= 1e-10 * abs(lhs)
    A = dense_siddon(N, len(theta), n_det, theta=theta)
    np.testing.assert_allclose(oracle.project_siddon(x, len(theta), n_det, theta=theta).ravel(), A @ x.ravel(),
                               rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.backproject_siddon(y, N, len(theta), theta=theta).ravel(),
                               A.T @ y.ravel(), rtol=0, atol=1e-12)

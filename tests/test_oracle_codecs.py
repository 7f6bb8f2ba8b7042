"""Pins of the oracle's quantizers: K-means (Alg. 5) and the
JPEG-style DCT codec, against the JPEG standard's printed table
(tests/golden), libjpeg's quality scaling (PIL), scipy's real orthonormal DCT,
brute-force 1-D clustering and the Lloyd fixed-point property."""
import io
import itertools
import json
import os

import numpy as np
import pytest
import scipy.fft

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ K-means
def test_kmeans_spec_example():
    """v = [0,0,1,1,10], K = 2 -> centres {0.5, 10}; decode
    [0.5,0.5,0.5,0.5,10] (the 1-D optimal 2-partition, reached from quantile init)."""
    cen, lab = oracle.kmeans_encode([0, 0, 1, 1, 10], 2, 10)
    assert sorted(cen.tolist()) == [0.5, 10.0]
    assert oracle.kmeans_decode(cen, lab).tolist() == [0.5, 0.5, 0.5, 0.5, 10.0]


def test_kmeans_single_cluster_is_mean():
    rng = np.random.default_rng(0)
    v = rng.standard_normal(1001).astype(np.float32)
    cen, lab = oracle.kmeans_encode(v, 1, 3)
    assert cen[0] == np.float32(np.mean(v.astype(np.float64)))
    assert not np.any(lab)


def test_kmeans_quantile_init_is_order_statistic():
    rng = np.random.default_rng(1)
    v = rng.random(777).astype(np.float32)
    K = 7
    cen, _ = oracle.kmeans_encode(v, K, 0)
    s = np.sort(v)
    assert np.array_equal(cen, s[[(2 * k + 1) * v.size // (2 * K) for k in range(K)]])


def test_kmeans_lloyd_fixed_point():
    """After Lloyd converges, every centre is the (fp32-rounded) mean of its cell and
    every element is assigned to a nearest centre."""
    rng = np.random.default_rng(2)
    v = np.concatenate([rng.normal(m, 0.05, 400) for m in (0.0, 0.3, 0.9, 1.7)]).astype(np.float32)
    cen, lab = oracle.kmeans_encode(v, 4, 200)
    for k in range(4):
        cell = v[lab == k]
        assert cell.size > 0
        assert cen[k] == np.float32(cell.astype(np.float64).mean())
    dist = np.abs(v[:, None].astype(np.float64) - cen[None, :].astype(np.float64))
    assert np.all(dist[np.arange(v.size), lab] <= dist.min(axis=1) + 1e-7)


def _brute_opt(v, K):
    s = np.sort(v.astype(np.float64))
    best = np.inf
    for cuts in itertools.combinations(range(1, len(s)), K - 1):
        parts = np.split(s, cuts)
        best = min(best, sum(((p - p.mean()) ** 2).sum() for p in parts))
    return best


def test_kmeans_vs_bruteforce_optimum():
    """1-D optimal clusters are contiguous in sorted order: brute force over all cut
    sets gives the optimum distortion.  Lloyd never beats it, and on well-separated
    data it reaches it."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        v = rng.integers(0, 10, rng.integers(4, 11)).astype(np.float32)
        for K in (1, 2, 3):
            cen, lab = oracle.kmeans_encode(v, K, 50)
            dist = float(((v.astype(np.float64) - cen[lab].astype(np.float64)) ** 2).sum())
            assert dist >= _brute_opt(v, K) - 1e-9
    v = np.array([0, 0.1, 0.05, 5, 5.1, 9.9, 10], np.float32)
    cen, lab = oracle.kmeans_encode(v, 3, 20)
    dist = float(((v.astype(np.float64) - cen[lab].astype(np.float64)) ** 2).sum())
    assert abs(dist - _brute_opt(v, 3)) < 1e-6


def test_kmeans_exact_when_levels_equal_k():
    v = np.repeat(np.array([0.25, 1.5, 2.0, 7.0], np.float32), 50)
    np.random.default_rng(4).shuffle(v)
    cen, lab = oracle.kmeans_encode(v, 4, 10)
    assert np.array_equal(oracle.kmeans_decode(cen, lab), v)


def test_kmeans_bits_per_element_matches_paper():
    """K = 16 -> 4 bits, K = 3 -> 2 bits, K = 32 -> 5 bits."""
    g = json.load(open(os.path.join(GOLD, "paper_values.json")))["kmeans_bits"]
    for K, bits in g["K_bits"]:
        assert int(np.ceil(np.log2(K))) == bits


# ------------------------------------------------------------------ DCT
def _annex_k():
    rows = [l.split() for l in open(os.path.join(GOLD, "jpeg_luminance_annex_k.txt"))
            if l.strip() and not l.startswith("#")]
    return np.array(rows, dtype=np.int32)


def test_dct_table_q50_is_annex_k():
    assert np.array_equal(oracle.dct_qtable(50), _annex_k())


def test_dct_tables_match_libjpeg_all_qualities():
    """IJG quality scaling reproduces libjpeg's luminance table for q = 1..100 (PIL)."""
    from PIL import Image
    img = Image.fromarray((np.random.default_rng(0).random((16, 16)) * 255).astype(np.uint8))
    for q in range(1, 101):
        b = io.BytesIO()
        img.save(b, "JPEG", quality=q)
        b.seek(0)
        ref = np.array(list(Image.open(b).quantization[0]), np.int32).reshape(8, 8)
        assert np.array_equal(oracle.dct_qtable(q), ref), q
    assert np.all(oracle.dct_qtable(100) == 1)


def _blocks(a):
    r, c = a.shape
    return a.reshape(r // 8, 8, c // 8, 8).transpose(0, 2, 1, 3).reshape(-1, 8, 8)


def test_integer_dct_close_to_orthonormal_dct():
    """With Q = 1 (q = 100) the coefficient is round(Y / 2^18) and Y / 2^18 is the
    integer approximation of the orthonormal 2-D DCT F of the level-shifted block:
    |coef - F| <= 0.5 + 0.2, and coef == round(F) for >= 99.9% of coefficients."""
    rng = np.random.default_rng(5)
    v = rng.random((64, 64)).astype(np.float32)
    v[0, 0], v[1, 1] = 0.0, 1.0  # min 0, max 1 -> p = rint(255 v)
    coef, mm = oracle.dct_encode(v, 100)
    p = np.clip(np.rint((v.astype(np.float64) - mm[0]) * 255.0 / (float(mm[1]) - mm[0])), 0, 255)
    F = np.stack([scipy.fft.dctn(b - 128.0, norm="ortho") for b in _blocks(p)])
    cf = coef.reshape(-1, 8, 8).astype(np.float64)
    assert np.max(np.abs(cf - F)) <= 0.7
    # the 4 guard bits kept between the passes round each 1-D coefficient to 1/16
    # (error std ~0.018), so on uniform-noise blocks ~2% of coefficients land across
    # a rounding boundary; a transposed / mis-scaled matrix would break both bounds
    assert np.mean(cf == np.round(F)) >= 0.97


def test_dct_decode_close_to_real_idct():
    """Decoded 8-bit samples equal clip(round(IDCT(coef Q)) + 128) for >= 99.5% of
    pixels and never differ by more than 1."""
    rng = np.random.default_rng(6)
    v = (rng.random((32, 48)) + np.linspace(0, 3, 48)[None, :]).astype(np.float32)
    for q in (25, 50, 75, 95):
        coef, mm = oracle.dct_encode(v, q)
        _, smp = oracle.dct_decode(coef, mm, 32, 48, q, return_samples=True)
        Q = oracle.dct_qtable(q).astype(np.float64)
        G = coef.reshape(-1, 8, 8) * Q
        ref = np.clip(np.round(np.stack([scipy.fft.idctn(g, norm="ortho") for g in G]) + 128), 0, 255)
        got = _blocks(smp.astype(np.float64))
        assert np.max(np.abs(got - ref)) <= 1
        assert np.mean(got == ref) >= 0.98


def test_dct_constant_vector_exact():
    v = np.full((16, 24), 3.25, np.float32)
    coef, mm = oracle.dct_encode(v, 50)
    assert not np.any(coef) and mm.tolist() == [3.25, 3.25]
    assert np.array_equal(oracle.dct_decode(coef, mm, 16, 24, 50), v)


def test_dct_roundtrip_quality100_ramp():
    """q = 100 on a smooth ramp -> round-trip RMSE <= 1% of the range."""
    v = np.add.outer(np.linspace(0, 1, 64), np.linspace(0, 2, 64)).astype(np.float32)
    coef, mm = oracle.dct_encode(v, 100)
    out = oracle.dct_decode(coef, mm, 64, 64, 100)
    assert np.sqrt(np.mean((out - v) ** 2)) <= 0.01 * (v.max() - v.min())
    # endpoints of the 8-bit map are exact
    assert out.min() >= mm[0] - 1e-6 and out.max() <= mm[1] + 1e-6


def test_dct_error_shrinks_with_quality():
    rng = np.random.default_rng(7)
    v = (np.add.outer(np.sin(np.arange(64) / 5), np.cos(np.arange(64) / 7)) +
         0.05 * rng.standard_normal((64, 64))).astype(np.float32)
    errs = []
    for q in (10, 30, 50, 75, 95):
        coef, mm = oracle.dct_encode(v, q)
        errs.append(np.sqrt(np.mean((oracle.dct_decode(coef, mm, 64, 64, q) - v) ** 2)))
    assert all(a > b for a, b in zip(errs, errs[1:]))


# ----------------------------------------------------------------- JPEG entropy coding (NEXT-2)
def _pil_jpeg(img, quality):
    from PIL import Image
    b = io.BytesIO()
    Image.fromarray(np.asarray(img, np.uint8), "L").save(b, "JPEG", quality=quality)
    return b.getvalue()


def _jpeg_parts(data):
    """Marker segments of a baseline JPEG file: DHT tables {(class, id): (bits, vals)} and
    the entropy-coded segment after SOS (up to the EOI marker)."""
    i, dht, ent = 2, {}, None
    while i < len(data):
        assert data[i] == 0xFF
        m = data[i + 1]
        if m == 0xD9:
            break
        L = data[i + 2] * 256 + data[i + 3]
        body = data[i + 4:i + 2 + L]
        if m == 0xC4:
            j = 0
            while j < len(body):
                tc, th = body[j] >> 4, body[j] & 15
                bits = np.frombuffer(body[j + 1:j + 17], np.uint8)
                nv = int(bits.sum())
                dht[(tc, th)] = (bits.copy(), np.frombuffer(body[j + 17:j + 17 + nv], np.uint8).copy())
                j += 17 + nv
        if m == 0xDA:
            s = i + 2 + L
            e = s
            while not (data[e] == 0xFF and data[e + 1] not in (0x00,) and not 0xD0 <= data[e + 1] <= 0xD7):
                e += 1
            ent = data[s:e]
            i = e
            continue
        i += 2 + L
    return dht, ent


def test_jpeg_huffman_tables_match_libjpeg():
    """The oracle's Annex K tables equal the DHT segments libjpeg (via PIL) writes."""
    dht, _ = _jpeg_parts(_pil_jpeg(np.zeros((8, 8)), 75))
    dc_bits, dc_val, ac_bits, ac_val = oracle.jpeg_tables()
    assert np.array_equal(dht[(0, 0)][0], dc_bits) and np.array_equal(dht[(0, 0)][1], dc_val)
    assert np.array_equal(dht[(1, 0)][0], ac_bits) and np.array_equal(dht[(1, 0)][1], ac_val)


def test_jpeg_hand_coded_blocks():
    """T.81 by hand: an all-zero block = DC category 0 ('00') + EOB ('1010') + two fill
    1s = 0x2B; DC +1 = '010' '1' + EOB = 0x5A; DC -1 = '010' '0' + EOB = 0x4A."""
    z = np.zeros(64, np.int16)
    assert oracle.jpeg_encode(z) == b"\x2b"
    z[0] = 1
    assert oracle.jpeg_encode(z) == b"\x5a"
    z[0] = -1
    assert oracle.jpeg_encode(z) == b"\x4a"


@pytest.mark.parametrize("quality,shape,seed", [(50, (16, 24), 1), (75, (32, 32), 2), (95, (8, 64), 3),
                                                (100, (24, 16), 4), (10, (40, 40), 5)])
def test_jpeg_reencodes_libjpeg_entropy_segment(quality, shape, seed):
    """libjpeg's entropy-coded segment decodes with the oracle and re-encodes to the same
    bytes (Huffman codes, category bits, ZRL/EOB, byte stuffing, fill bits)."""
    rng = np.random.default_rng(seed)
    img = rng.integers(0, 256, size=shape)
    img[: shape[0] // 2] = np.clip(img[: shape[0] // 2] // 8 + 100, 0, 255)  # smooth + noisy halves
    _, ent = _jpeg_parts(_pil_jpeg(img, quality))
    nb = shape[0] * shape[1] // 64
    coef = oracle.jpeg_decode(ent, nb, 0)
    assert oracle.jpeg_encode(coef, 0) == ent
    if quality >= 95:  # long noisy streams: byte stuffing is exercised
        assert b"\xff\x00" in ent


def test_jpeg_zigzag_pinned_by_libjpeg_basis_images():
    """Figure A.6 and the natural layout: libjpeg (quality 100, all-ones table) codes the
    DCT basis image of vertical frequency a, horizontal frequency b with its dominant
    coefficient at natural index 8a + b of the oracle's decode."""
    x = np.arange(8)
    for a in range(8):
        for b in range(8):
            if a == b == 0:
                continue
            basis = np.outer(np.cos((2 * x + 1) * a * np.pi / 16), np.cos((2 * x + 1) * b * np.pi / 16))
            img = np.clip(np.rint(128 + 100 * basis), 0, 255)
            _, ent = _jpeg_parts(_pil_jpeg(img, 100))
            c = oracle.jpeg_decode(ent, 1, 0).astype(np.int64)
            ac = c.copy()
            ac[0] = 0
            assert int(np.argmax(np.abs(ac))) == 8 * a + b, (a, b)
    z = oracle.jpeg_zigzag()
    assert sorted(z.tolist()) == list(range(64)) and z[1] == 1 and z[2] == 8 and z[63] == 63


@pytest.mark.parametrize("restart", [0, 1, 3, 8])
def test_jpeg_restart_roundtrip_and_markers(restart):
    rng = np.random.default_rng(10 + restart)
    nb = 45
    c = (rng.integers(-40, 41, size=nb * 64) * (rng.random(nb * 64) < 0.2)).astype(np.int16)
    c[::64] = rng.integers(-1024, 1017, size=nb)  # DC differences up to 11 bits
    s = oracle.jpeg_encode(c, restart)
    assert np.array_equal(oracle.jpeg_decode(s, nb, restart), c)
    # RSTm markers: one per interval boundary, m cycling 0..7 (F.1.4.4 / B.2.1)
    marks = [s[i + 1] for i in range(len(s) - 1) if s[i] == 0xFF and 0xD0 <= s[i + 1] <= 0xD7]
    n_int = 0 if restart == 0 else (nb + restart - 1) // restart - 1
    assert marks == [0xD0 + (k % 8) for k in range(n_int)]
    # every 0xFF data byte is stuffed
    for i in range(len(s) - 1):
        if s[i] == 0xFF:
            assert s[i + 1] == 0x00 or 0xD0 <= s[i + 1] <= 0xD7
    # a restart resets the DC predictor: interval k's first block codes its DC absolutely,
    # so each interval decodes alone
    if restart:
        parts = s.split(b"\xff\xd0")[0] if n_int else s
        first = oracle.jpeg_decode(parts, min(restart, nb), restart)
        assert np.array_equal(first, c[:64 * min(restart, nb)])


def test_jpeg_extreme_values_and_runs():
    """AC +-1023 (category 10), DC jumps of 2040 (category 11), runs of 15, 16, 17 and 62
    zeros (ZRL), a non-zero last coefficient (no EOB), an all-zero block."""
    zz = oracle.jpeg_zigzag()
    blocks = []
    b = np.zeros(64, np.int16); b[0] = -1024; b[zz[1]] = 1023; b[zz[17]] = -1023; blocks.append(b)
    b = np.zeros(64, np.int16); b[0] = 1016; b[zz[63]] = 5; blocks.append(b)
    b = np.zeros(64, np.int16); b[zz[16]] = 1; b[zz[33]] = -2; b[zz[51]] = 3; blocks.append(b)
    blocks.append(np.zeros(64, np.int16))
    b = np.zeros(64, np.int16); b[zz[63]] = -1; blocks.append(b)
    c = np.concatenate(blocks)
    for r in (0, 2):
        assert np.array_equal(oracle.jpeg_decode(oracle.jpeg_encode(c, r), len(blocks), r), c)
    bad = np.zeros(64, np.int16); bad[1] = 1024  # outside the baseline AC categories
    with pytest.raises(ValueError):
        oracle.jpeg_encode(bad)
    with pytest.raises(ValueError):
        oracle.jpeg_decode(b"\x2b\x00", 1, 0)  # trailing garbage

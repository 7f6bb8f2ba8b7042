"""Seeded synthetic inputs (no method arithmetic): the NEXT-1 paper-shaped phantom."""
import numpy as np

from paper_2410_06106_b200 import synth


def test_three_level_phantom_levels_and_support():
    """PAPER.md:343 'three distinct gray levels': sampled at pixel centres the phantom
    takes exactly {0, 0.5, 1} and lies inside the inscribed circle (all rays see it)."""
    for seed in (7001, 7002, 7003):
        e = synth.three_level_phantom(256, seed)
        img = synth.rasterize(e, 256, supersample=1)
        assert set(np.unique(img)) == {0.0, 0.5, 1.0}
        xs, ys = synth.pixel_centres(256)
        r = np.hypot(xs[None, :], ys[:, None])
        assert np.all(img[r > 128] == 0)
        assert 5 <= len(e) - 1 <= 8


def test_paper_sinogram_noise_is_nsd_of_peak():
    """sigma = NSD x max(d_clean)."""
    e = synth.three_level_phantom(64, 1)
    d = synth.ellipse_sinogram(e, synth.default_angles(50), 91)
    noisy = synth.add_noise(d, 0.0243, 5)
    assert abs(np.std(noisy - d) / d.max() - 0.0243) < 0.002

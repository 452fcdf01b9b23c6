"""The seeded input generator (synth/): determinism and the noise model's moments
(P:273-281 with the D415 parameters of P:350; SPEC acceptance #5 moment checks)."""
import numpy as np

import synth


def test_deterministic_and_distinct():
    a = synth.make_pair("B", 3)
    b = synth.make_pair("B", 3)
    c = synth.make_pair("B", 4)
    assert all(np.array_equal(x, y, equal_nan=True) for x, y in zip(a, b))
    assert not np.array_equal(a[0], c[0])


def test_noise_moments():
    rng = synth.rng_for(0, 99)
    clean = np.full(1_000_000, 100.0)
    out = synth.apply_noise(clean, rng)
    k, th, mu, sg = synth.NOISE_K, synth.NOISE_THETA, synth.NOISE_MU, synth.NOISE_SIGMA
    mean = k * th * 100 + mu
    var = k * th * th * 100 ** 2 + sg ** 2
    assert abs(out.mean() - mean) / mean < 0.01
    assert abs(out.var() - var) / var < 0.03
    n = synth.apply_noise(np.zeros(1_000_000), rng)
    assert abs((n < 0).mean() - 0.61) < 0.01


def test_speckle_disparity_range_fits_configs():
    for name in ("B", "C", "D"):
        cfg = synth.CONFIGS[name]
        _, _, gt = synth.make_pair(name, 0)
        g = gt[~np.isnan(gt)]
        assert g.min() > cfg.min_disp and g.max() < cfg.min_disp + cfg.num_disp - 1


def test_shift_pair_exact():
    L, R, gt = synth.shift_pair(64, 48, 7)
    assert np.array_equal(R[:, :-7], L[:, 7:]) and (gt == 7).all()

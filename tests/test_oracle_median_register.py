"""Pins for oracle O9 (median, "median filtering", SPEC S:342-347,
reading c20) and O10 (depth registration, reading c21)."""
import numpy as np
import pytest

import oracle
import synth


def _p(W, H, k):
    return oracle.Params(width=W, height=H, num_disp=16, census_w=3, census_h=3, median_ksize=k)


def _median_numpy(dl, mask, k):
    """Independent restatement: gather the valid window values, sort, lower median."""
    H, W = dl.shape
    out = dl.copy()
    r = k // 2
    for y in range(H):
        for x in range(W):
            if k == 0 or (mask[y, x] & 7):
                continue
            v = [dl[yy, xx] for yy in range(max(0, y - r), min(H, y + r + 1))
                 for xx in range(max(0, x - r), min(W, x + r + 1)) if not (mask[yy, xx] & 7)]
            out[y, x] = np.sort(np.array(v, np.float32))[(len(v) - 1) // 2]
    return out


def test_median_ksize0_identity():
    rng = np.random.default_rng(0)
    dl = rng.uniform(0, 20, (6, 7)).astype(np.float32)
    mask = rng.integers(0, 2, (6, 7)).astype(np.uint8)
    assert np.array_equal(oracle.median(_p(7, 6, 0), dl, mask), dl)


def test_median_removes_single_spike():
    """a single-pixel spike in a constant plane is removed at ksize 3."""
    dl = np.full((9, 9), 10.0, np.float32)
    dl[4, 4] = 30.0
    out = oracle.median(_p(9, 9, 3), dl, np.zeros((9, 9), np.uint8))
    assert (out == 10.0).all()


def test_median_half_invalid_window_and_lower_median():
    """half-invalid window -> median of the valid half; an even count
    takes the lower of the two middle values (reading c20)."""
    dl = np.array([[1, 2, 9], [3, 4, 9], [9, 9, 9]], np.float32)
    mask = np.array([[0, 0, 2], [0, 0, 4], [1, 2, 4]], np.uint8)   # 4 valid: 1,2,3,4
    out = oracle.median(_p(3, 3, 3), dl, mask)
    assert out[1, 1] == 2.0                      # lower median of {1,2,3,4}
    assert out[0, 2] == 9.0 and out[2, 0] == 9.0  # invalid pixels keep their value
    assert out[0, 0] == 2.0                      # window {1,2,3,4} clipped at the corner


@pytest.mark.parametrize("k", [3, 5])
def test_median_matches_numpy(k):
    rng = np.random.default_rng(k)
    for _ in range(20):
        H, W = rng.integers(1, 12), rng.integers(1, 12)
        dl = rng.integers(0, 6, (H, W)).astype(np.float32) + rng.choice([0.0, 0.25, 0.5], (H, W)).astype(np.float32)
        mask = (rng.random((H, W)) < 0.3).astype(np.uint8) * rng.choice([1, 2, 4, 8], (H, W)).astype(np.uint8)
        assert np.array_equal(oracle.median(_p(W, H, k), dl, mask), _median_numpy(dl, mask, k))


def test_median_in_pipeline_keeps_a_plane():
    """compute() with median 3 on the +7 shifted pair: valid interior disparities stay 7."""
    left, right, _ = synth.shift_pair(64, 48, 7, frame_idx=0)
    d = synth.CONFIGS["A"].params_dict()
    o0 = oracle.compute(oracle.Params(**d), left, right)
    o3 = oracle.compute(oracle.Params(**d, median_ksize=3), left, right)
    v = (o0["mask"] == 0) & (o3["mask"] == 0)
    assert v.mean() > 0.7
    assert (np.abs(o3["disp"][v] - 7.0) < 0.5).mean() >= 0.99
    # smoothing: the median is no farther from the true plane than the raw map
    assert np.abs(o3["disp"][v] - 7.0).mean() <= np.abs(o0["disp"][v] - 7.0).mean()
    # the median only changes values, never validity before the depth stage
    assert np.array_equal(o0["mask"] & 7, o3["mask"] & 7)


# ------------------------------------------------------------------ O10
CAM = (40, 30, 100.0, 100.0, 19.5, 14.5)
EYE = np.eye(3, dtype=np.float32)


def test_register_identity():
    """rgb_cam == ir_cam -> output equals input on valid pixels."""
    rng = np.random.default_rng(1)
    z = rng.uniform(0.3, 3.0, (30, 40)).astype(np.float32)
    z[rng.random((30, 40)) < 0.2] = np.nan
    out = oracle.register(CAM, CAM, EYE, [0, 0, 0], z)
    assert np.array_equal(np.isnan(out), np.isnan(z))
    v = ~np.isnan(z)
    assert np.array_equal(out[v], z[v])


def test_register_translation_shifts_wall():
    """rgb_cam translated +x by b -> a wall at depth z shifts by fx*b/z px
    (here fx*b/z = 100 * 0.05 / 1.0 = 5 px to the left)."""
    z = np.ones((30, 40), np.float32)
    out = oracle.register(CAM, CAM, EYE, [-0.05, 0, 0], z)
    assert (out[:, :35] == 1.0).all()
    assert np.isnan(out[:, 35:]).all()


def test_register_nearer_surface_wins():
    """two samples on one target pixel -> the nearer depth."""
    z = np.full((30, 40), np.nan, np.float32)
    z[5, 10] = 1.0        # shifts by 5 px  -> target (5, 5)
    z[5, 7] = 2.5         # shifts by 2 px  -> target (5, 5)
    out = oracle.register(CAM, CAM, EYE, [-0.05, 0, 0], z)
    assert out[5, 5] == 1.0
    assert np.isnan(out).sum() == out.size - 1


def test_register_matches_fp64_projection():
    """Random rigid motion and a larger RGB camera: the oracle's fp32 target
    pixels and depths agree with an independent fp64 projection wherever no
    source lands within 1e-3 px of a rounding boundary."""
    rng = np.random.default_rng(7)
    ir = (64, 48, 120.0, 121.0, 31.5, 23.5)
    rgb = (96, 72, 180.0, 181.0, 47.0, 35.0)
    ang = 0.05
    R = np.array([[np.cos(ang), 0, np.sin(ang)], [0, 1, 0], [-np.sin(ang), 0, np.cos(ang)]], np.float32)
    t = np.array([-0.015, 0.002, 0.001], np.float32)
    z = rng.uniform(0.4, 2.0, (48, 64)).astype(np.float32)
    z[rng.random((48, 64)) < 0.1] = np.nan
    out = oracle.register(ir, rgb, R, t, z)
    ref = np.full((72, 96), np.inf)
    amb = np.zeros((72, 96), bool)
    ys, xs = np.nonzero(~np.isnan(z))
    zz = z[ys, xs].astype(np.float64)
    a = (xs - ir[4]) * zz / ir[2]
    b = (ys - ir[5]) * zz / ir[3]
    P = R.astype(np.float64) @ np.stack([a, b, zz]) + t.astype(np.float64)[:, None]
    u = P[0] / P[2] * rgb[2] + rgb[4] + 0.5
    v = P[1] / P[2] * rgb[3] + rgb[5] + 0.5
    for uu, vv, Z in zip(u, v, P[2]):
        iu, iv = int(np.floor(uu)), int(np.floor(vv))
        near = min(uu - np.floor(uu), np.ceil(uu) - uu, vv - np.floor(vv), np.ceil(vv) - vv) < 1e-3
        for du in (-1, 0, 1):
            for dv in (-1, 0, 1):
                ju, jv = iu + du, iv + dv
                if near and 0 <= ju < 96 and 0 <= jv < 72:
                    amb[jv, ju] = True
        if 0 <= iu < 96 and 0 <= iv < 72:
            ref[iv, iu] = min(ref[iv, iu], Z)
    ref[np.isinf(ref)] = np.nan
    ok = ~amb
    assert ok.mean() > 0.9
    assert np.array_equal(np.isnan(out[ok]), np.isnan(ref[ok]))
    f = ok & ~np.isnan(ref)
    assert f.sum() > 1000
    assert np.abs(out[f] - ref[f]).max() <= 1e-5 * np.abs(ref[f]).max()

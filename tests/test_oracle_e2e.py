"""End-to-end pins for the oracle (acceptance #4; BASELINE.json north_star)."""
import numpy as np
import pytest

import oracle
import synth


def _pA(**kw):
    d = synth.CONFIGS["A"].params_dict()
    d.update(kw)
    return oracle.Params(**d)


def _interior(p, s):
    R, Q = p.census_w // 2, p.census_h // 2
    m = np.zeros((p.height, p.width), bool)
    m[Q:p.height - Q, R + s:p.width - R] = True
    return m


@pytest.mark.parametrize("frame", [0, 1, 2])
def test_integer_shift_recovered(frame):
    """S:371 / acceptance #4: +7 px shift -> >= 99% of interior pixels have d* = 7,
    and the LR check keeps >= 99% of them; dr = 7 too."""
    left, right, _ = synth.shift_pair(64, 48, 7, frame_idx=frame)
    p = _pA()
    o = oracle.compute(p, left, right)
    inner = _interior(p, 7)
    assert (o["dstar_l"][inner] == 7).mean() >= 0.99
    valid = o["mask"][inner] == 0
    assert (o["dstar_l"][inner][valid] == 7).all()
    # LR on the interior minus 2 columns: right pixels xr < R + 2 see S_R built from
    # left pixels whose costs are nb at every d but 0 (reading c10 near the border).
    inner_lr = inner.copy()
    inner_lr[:, :p.census_w // 2 + 7 + 2] = False
    lr_fail = (o["mask"][inner_lr] & oracle.MASK_LR) != 0
    assert lr_fail.mean() <= 0.01
    R, Q = p.census_w // 2, p.census_h // 2
    assert (o["dstar_r"][Q:-Q, R + 2:p.width - R - 7] == 7).mean() >= 0.99


def test_fronto_parallel_plane_depth():
    """BJ: a fronto-parallel plane at integer shift s -> median depth f*b/s."""
    p = _pA()
    for s in (5, 7, 9):
        left, right, _ = synth.shift_pair(64, 48, s, frame_idx=10 + s)
        o = oracle.compute(p, left, right)
        fb = float(np.float32(p.focal_px)) * float(np.float32(p.baseline_m))
        assert np.nanmedian(o["depth"]) == pytest.approx(fb / s, rel=1e-12)


def test_fractional_shift_subpixel():
    """6.5 px bilinear shift -> median |d - 6.5| <= 0.25 on valid interior."""
    left, right, _ = synth.shift_pair(64, 48, 6.5, frame_idx=3)
    p = _pA()
    o = oracle.compute(p, left, right)
    inner = _interior(p, 7)
    v = inner & (o["mask"] == 0)
    assert v.sum() > 0.5 * inner.sum()
    assert np.median(np.abs(o["disp"][v] - 6.5)) <= 0.25


def test_textureless_mostly_invalid():
    """textureless frames -> >= 99% INVALID (uniqueness kills flat cost)."""
    p = _pA()
    z = np.zeros((48, 64), np.uint8)
    o = oracle.compute(p, z, z)
    assert (o["mask"] != 0).mean() >= 0.99


def test_brightness_invariance():
    """compute_depth(L + c, R + c) == compute_depth(L, R) without saturation."""
    rng = np.random.default_rng(1)
    T = rng.integers(0, 200, size=(48, 72), dtype=np.uint8)
    L, R = T[:, :64].copy(), T[:, 7:71].copy()
    p = _pA()
    a = oracle.compute(p, L, R)
    b = oracle.compute(p, L + np.uint8(40), R + np.uint8(40))
    for k in ("dstar_l", "dstar_r", "mask", "dl", "dr"):
        assert np.array_equal(a[k], b[k]), k


def test_monotone_invalidation():
    """raising uniqueness or lowering lr_max_diff never turns INVALID valid."""
    left, right, _ = synth.make_pair("A", 4)
    prev = None
    for u in (0, 10, 30):
        bad = oracle.compute(_pA(uniqueness=u), left, right)["mask"] != 0
        if prev is not None:
            assert (bad >= prev).all()
        prev = bad
    prev = None
    for lr in (4.0, 1.0, 0.5, 0.1):
        bad = oracle.compute(_pA(lr_max_diff=lr), left, right)["mask"] != 0
        if prev is not None:
            assert (bad >= prev).all()
        prev = bad


def test_disparity_bounds_and_speckle_scene():
    """valid dl in [min_disp - 0.5, max_disp - 0.5); on a B-shaped speckle
    scene (cropped) most valid disparities are within 1 px of the ground truth."""
    cfg = synth.CONFIGS["B"]
    left, right, gt = synth.make_pair("B", 0)
    d = cfg.params_dict()
    d.update(width=320, height=96)
    p = oracle.Params(**d)
    L = np.ascontiguousarray(left[100:196, 200:520])
    R = np.ascontiguousarray(right[100:196, 200:520])
    o = oracle.compute(p, L, R)
    v = o["mask"] == 0
    assert v.mean() > 0.5
    dv = o["disp"][v]
    assert (dv >= p.min_disp - 0.5).all() and (dv < p.min_disp + p.num_disp - 0.5).all()
    g = gt[100:196, 200:520][v]
    ok = ~np.isnan(g)
    assert (np.abs(dv[ok] - g[ok]) < 1.0).mean() > 0.9
    assert np.isnan(o["disp"][~v]).all() and np.isnan(o["depth"][~v]).all()

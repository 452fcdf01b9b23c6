"""Pins for oracle O4-O8 (WTA + uniqueness, sub-pixel, right view, LR, depth);
PAPER.md P:289, readings c8-c14."""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _S(costs):
    return np.array(costs, np.uint32).reshape(1, 1, -1)


def _p(D, **kw):
    base = dict(width=1, height=1, num_disp=D, census_w=1, census_h=1)
    base.update(kw)
    return oracle.Params(**base)


def test_golden_wta_examples():
    g = json.load(open(os.path.join(GOLD, "wta_subpixel.json")))
    for case in g["wta"]:
        p = _p(len(case["costs"]), uniqueness=case["uniqueness"], subpixel=0)
        ds, m, dl = oracle.wta_left(p, _S(case["costs"]))
        assert int(ds[0, 0]) == case["dstar"], case
        assert bool(m[0, 0] & oracle.MASK_UNIQUE) == case["unique_fail"], case
    for case in g["subpixel"]:
        p = _p(len(case["costs"]), uniqueness=-1, subpixel=1)
        ds, m, dl = oracle.wta_left(p, _S(case["costs"]))
        assert int(ds[0, 0]) == case["dstar"] and float(dl[0, 0]) == case["disp"], case


@pytest.mark.parametrize("m,j", [(4, 1), (4, -1), (8, 3), (2, 1), (16, -7), (4, 2)])
def test_subpixel_exact_parabola(m, j):
    """Closed form: S(d) = (m(d-k) - j)^2 + c is a parabola with vertex k + j/m, so
    the quadratic fit must return exactly k + j/m (|j/m| <= 1/2, m a power of 2)."""
    D, k, c = 12, 5, 7
    costs = [(m * (d - k) - j) ** 2 + c for d in range(D)]
    ds, _, dl = oracle.wta_left(_p(D, uniqueness=-1, min_disp=3), _S(costs))
    best = int(np.argmin(costs))
    assert int(ds[0, 0]) == best
    assert float(dl[0, 0]) == 3 + k + j / m


def test_subpixel_offset_range_and_ends():
    """Offset in (-0.5, 0.5] at an interior smallest argmin; 0 at the range ends."""
    rng = np.random.default_rng(2)
    p = oracle.Params(width=64, height=64, num_disp=24, census_w=1, census_h=1, uniqueness=-1)
    S = rng.integers(0, 500, size=(64, 64, 24)).astype(np.uint32)
    ds, _, dl = oracle.wta_left(p, S)
    off = dl - ds.astype(np.float32)
    assert (off > -0.5).all() and (off <= 0.5).all()
    ends = (ds == 0) | (ds == 23)
    assert (off[ends] == 0).all()
    assert np.array_equal(ds, np.argmin(S, axis=2))


def test_uniqueness_monotone_in_ratio():
    """raising the uniqueness ratio never turns an invalid pixel valid."""
    rng = np.random.default_rng(4)
    S = rng.integers(0, 100, size=(32, 32, 16)).astype(np.uint32)
    prev = None
    for u in [0, 5, 10, 20, 50, 100]:
        p = oracle.Params(width=32, height=32, num_disp=16, census_w=1, census_h=1, uniqueness=u)
        bad = (oracle.wta_left(p, S)[1] & oracle.MASK_UNIQUE) != 0
        if prev is not None:
            assert (bad | ~prev).all() and (bad >= prev).all()
        prev = bad


def test_depth_examples():
    """f=100, b=0.055, d=10 -> 0.55 m; d=0 -> INVALID; z*d = f*b."""
    p = oracle.Params(width=3, height=1, num_disp=16, census_w=1, census_h=1,
                      lr_max_diff=-1, focal_px=100.0, baseline_m=0.055)
    dl = np.array([[10.0, 0.0, 2.5]], np.float32)
    m, disp, z = oracle.lr_depth(p, dl, dl, np.zeros((1, 3), np.uint8), np.zeros((1, 3), np.uint8))
    fb = float(np.float32(100.0)) * float(np.float32(0.055))
    assert abs(z[0, 0] - 0.55) < 1e-7 and z[0, 0] == fb / 10.0
    assert np.isnan(z[0, 1]) and np.isnan(disp[0, 1]) and m[0, 1] == oracle.MASK_NONPOS
    assert z[0, 2] * 2.5 == pytest.approx(fb, rel=1e-15)


def test_lr_cases():
    """dr all INVALID -> all INVALID; lr = inf -> dl wherever the lookup
    lands in bounds; a consistent pair survives."""
    W = 20
    p = oracle.Params(width=W, height=1, num_disp=8, census_w=1, census_h=1, lr_max_diff=1.0)
    dl = np.full((1, W), 3.25, np.float32)
    dr = np.full((1, W), 3.0, np.float32)
    ok = np.zeros((1, W), np.uint8)
    m, disp, _ = oracle.lr_depth(p, dl, dr, np.ones((1, W), np.uint8), ok)
    assert (m & oracle.MASK_LR).all()
    m, disp, _ = oracle.lr_depth(p, dl, dr, ok, ok)
    xr = np.arange(W) - 3
    assert ((m == 0) == (xr >= 0)).all() and (disp[0, 3:] == 3.25).all()
    p_inf = oracle.Params(width=W, height=1, num_disp=8, census_w=1, census_h=1, lr_max_diff=1e30)
    m, disp, _ = oracle.lr_depth(p_inf, dl, dr + 5, ok, ok)
    assert ((m == 0) == (xr >= 0)).all()
    p_tight = oracle.Params(width=W, height=1, num_disp=8, census_w=1, census_h=1, lr_max_diff=0.2)
    m, _, _ = oracle.lr_depth(p_tight, dl, dr, ok, ok)
    assert (m & oracle.MASK_LR).all()
    # half-up rounding (reading c11): dl = 3.5 looks up x - 4
    dl2 = np.full((1, W), 3.5, np.float32)
    dr2 = np.zeros((1, W), np.float32)
    dr2[0, 10 - 4] = 3.5
    m, _, _ = oracle.lr_depth(p, dl2, dr2, ok, ok)
    assert m[0, 10] == 0 and (m[0, 4:10] & oracle.MASK_LR).all()


def test_lr_skips_border_and_unique_failures():
    W = 10
    p = oracle.Params(width=W, height=1, num_disp=8, census_w=1, census_h=1, lr_max_diff=1.0)
    dl = np.full((1, W), 2.0, np.float32)
    pre = np.zeros((1, W), np.uint8)
    pre[0, 5] = oracle.MASK_BORDER
    pre[0, 6] = oracle.MASK_UNIQUE
    m, _, _ = oracle.lr_depth(p, dl, dl, np.ones((1, W), np.uint8), pre)
    assert m[0, 5] == oracle.MASK_BORDER and m[0, 6] == oracle.MASK_UNIQUE


def test_right_view_mirrors_left_view_without_smoothing():
    """Reading c10 (R1) pinned where it has a closed form: with P1 = P2 = 0, S =
    paths*C, so the re-indexed right view of (L, R) equals the mirrored left view
    of (flip R, flip L) wherever every disparity is defined.  Images use distinct
    values (no census ties) so mirroring permutes/complements census bits
    identically on both sides and Hamming distances are preserved."""
    W, H, D = 16, 12, 4
    rng = np.random.default_rng(21)
    vals = rng.permutation(256)[:W * H].astype(np.uint8)
    L = vals.reshape(H, W)
    R = np.roll(L, -2, axis=1).copy()
    R[:, -2:] = rng.permutation(np.setdiff1d(np.arange(256), vals))[:2 * H].reshape(H, 2)
    p = oracle.Params(width=W, height=H, num_disp=D, census_w=3, census_h=3,
                      p1=0, p2=0, paths=4, uniqueness=10)
    o = oracle.compute(p, L, R)
    f = oracle.compute(p, R[:, ::-1].copy(), L[:, ::-1].copy())
    keep = slice(0, W - D)          # xr + (D-1) < W - 1: every d defined, incl. neighbours
    assert np.array_equal(o["dstar_r"][:, keep], f["dstar_l"][:, ::-1][:, keep])
    assert np.array_equal(o["dr"][:, keep], f["dl"][:, ::-1][:, keep])
    mr = o["mask_r"][:, keep]
    ml = oracle.wta_left(p, oracle.sgm(p, oracle.cost(p, oracle.census(p, R[:, ::-1].copy()),
                                                      oracle.census(p, L[:, ::-1].copy()))))[1]
    assert np.array_equal(mr, ml[:, ::-1][:, keep])


def test_right_view_undefined_disparities():
    """O6: S_R(xr, d) is defined only for xr + delta(d) < W; the rightmost pixel
    sees only d = 0 (min_disp = 0)."""
    W, D = 8, 4
    S = np.arange(W * D, dtype=np.uint32)[::-1].reshape(1, W, D).copy()
    p = oracle.Params(width=W, height=1, num_disp=D, census_w=1, census_h=1, uniqueness=-1)
    ds, m, dr = oracle.wta_right(p, S)
    assert ds[0, W - 1] == 0 and m[0, W - 1] == 0
    for xr in range(W):
        cand = [(S[0, xr + d, d], d) for d in range(D) if xr + d < W]
        assert ds[0, xr] == min(cand)[1]
    p2 = oracle.Params(width=W, height=1, num_disp=D, min_disp=W, census_w=1, census_h=1)
    ds, m, _ = oracle.wta_right(p2, S)
    assert (ds == -1).all() and (m & oracle.MASK_BORDER).all()

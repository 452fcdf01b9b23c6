"""Pins for oracle O1 (CSCT census) and O2 (Hamming cost)."""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_golden_3x3_cases():
    """S:294-295 examples plus hand-enumerated ramps (fixture census_3x3.json)."""
    g = json.load(open(os.path.join(GOLD, "census_3x3.json")))
    p = oracle.Params(width=3, height=3, census_w=3, census_h=3)
    for case in g["cases"]:
        img = np.array(case["image"], np.uint8)
        c = oracle.census(p, img)
        assert int(c[1, 1]) == case["center_sig"], case
        border = np.ones((3, 3), bool)
        border[1, 1] = False
        assert (c[border] == 0).all()


@pytest.mark.parametrize("cw,ch", [(3, 3), (5, 5), (7, 7), (9, 7), (11, 11)])
def test_single_bright_pixel_sets_its_pair_bit(cw, ch):
    """S:295 generalised: a lone bright pixel at row-major window index j sets bit j
    when j < nb (it is p_a of pair j); when j > nb it is p_b of pair N-1-j, whose
    comparison is then false, so the signature is 0.  A lone DARK pixel at j > nb
    sets bit N-1-j."""
    nb = (cw * ch) // 2
    N = cw * ch
    p = oracle.Params(width=cw, height=ch, census_w=cw, census_h=ch)
    for j in range(N):
        if j == nb:
            continue
        img = np.full((ch, cw), 50, np.uint8)
        img[j // cw, j % cw] = 200
        sig = int(oracle.census(p, img)[ch // 2, cw // 2])
        assert sig == ((1 << j) if j < nb else 0)
        img = np.full((ch, cw), 200, np.uint8)
        img[j // cw, j % cw] = 50
        sig = int(oracle.census(p, img)[ch // 2, cw // 2])
        assert sig == ((1 << (N - 1 - j)) if j > nb else 0)


def test_constant_image_is_zero():
    """strict > yields 0 on ties."""
    p = oracle.Params(width=40, height=30, census_w=9, census_h=7)
    assert (oracle.census(p, np.full((30, 40), 77, np.uint8)) == 0).all()


def test_brightness_offset_invariance():
    """census(I) == census(I + c) without saturation."""
    rng = np.random.default_rng(5)
    p = oracle.Params(width=50, height=40, census_w=9, census_h=7)
    I = rng.integers(0, 200, size=(40, 50), dtype=np.uint8)
    assert np.array_equal(oracle.census(p, I), oracle.census(p, I + np.uint8(55)))


@pytest.mark.parametrize("cw,ch", [(3, 3), (5, 5), (9, 7), (11, 11)])
def test_rotation_by_180_complements(cw, ch):
    """Centre symmetry: rotating the image by 180 deg swaps p_a and p_b of every
    pair, so with no ties the signature at the rotated pixel is the complement."""
    W, H = 16, 16
    rng = np.random.default_rng(cw * 100 + ch)
    I = rng.permutation(256).astype(np.uint8).reshape(H, W)      # all values distinct
    p = oracle.Params(width=W, height=H, census_w=cw, census_h=ch)
    c = oracle.census(p, I)
    c_rot = oracle.census(p, I[::-1, ::-1].copy())[::-1, ::-1]
    R, Q = cw // 2, ch // 2
    full = np.uint64((1 << ((cw * ch) // 2)) - 1)
    inner = (slice(Q, H - Q), slice(R, W - R))
    assert np.array_equal(c_rot[inner], (~c[inner]) & full)


def test_border_pixels_are_zero():
    rng = np.random.default_rng(6)
    p = oracle.Params(width=30, height=20, census_w=9, census_h=7)
    c = oracle.census(p, rng.integers(0, 256, size=(20, 30), dtype=np.uint8))
    assert (c[:3] == 0).all() and (c[-3:] == 0).all()
    assert (c[:, :4] == 0).all() and (c[:, -4:] == 0).all()
    assert (c[3:-3, 4:-4] != 0).mean() > 0.99


def test_cost_identical_views_zero_plane():
    """cl == cr -> the d=0 plane is zero on valid pixels."""
    rng = np.random.default_rng(8)
    p = oracle.Params(width=48, height=32, num_disp=16, census_w=5, census_h=5)
    I = rng.integers(0, 256, size=(32, 48), dtype=np.uint8)
    c = oracle.census(p, I)
    C = oracle.cost(p, c, c)
    assert (C[2:-2, 2:-2, 0] == 0).all()
    assert (C <= p.nbits).all()


@pytest.mark.parametrize("s", [0, 3, 5, 7])
def test_cost_shift_plane_zero(s):
    """right = left shifted +s -> the d=s plane is zero on the interior,
    every other plane is > 0 somewhere; out-of-range entries cost nb (reading c3)."""
    left, right, _ = synth.shift_pair(64, 48, s, frame_idx=s)
    p = oracle.Params(width=64, height=48, num_disp=16, census_w=5, census_h=5)
    C = oracle.cost(p, oracle.census(p, left), oracle.census(p, right))
    R = Q = 2
    inner = C[Q:-Q, R + s:-R]
    assert (inner[:, :, s] == 0).all()
    for d in range(16):
        if d != s:
            assert (C[Q:-Q, R + d:-R, d] > 0).any()
    for d in range(16):                        # x - d < R -> invalid -> nb
        assert (C[:, :R + d, d] == p.nbits).all()
    assert (C[:Q] == p.nbits).all() and (C[:, -R:] == p.nbits).all()


def test_cost_is_popcount_of_xor():
    """Spot check of O2 against Python's own bit counting on random census pairs."""
    rng = np.random.default_rng(9)
    p = oracle.Params(width=40, height=20, num_disp=8, census_w=5, census_h=5)
    L = rng.integers(0, 256, size=(20, 40), dtype=np.uint8)
    R = rng.integers(0, 256, size=(20, 40), dtype=np.uint8)
    cl, cr = oracle.census(p, L), oracle.census(p, R)
    C = oracle.cost(p, cl, cr)
    for d in range(8):
        for x in range(2 + d, 38):
            assert (C[2:-2, x, d] == [bin(int(a) ^ int(b)).count("1")
                                       for a, b in zip(cl[2:-2, x], cr[2:-2, x - d])]).all()

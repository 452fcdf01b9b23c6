"""Pins for the SGBM cost (oracle O2b, reading c19).

CB(x,y,d) = sum over the bw x bh block of C~(x+u, y+v, d), with C~ = the
per-pixel Hamming cost (O2) inside the image and nb outside it.
"""
import numpy as np
import pytest

import oracle
import synth
from tests.brute_sgm import aggregate_bruteforce


def _p(W, H, D, bw, bh, cw=3, ch=3, **kw):
    return oracle.Params(width=W, height=H, num_disp=D, census_w=cw, census_h=ch,
                         block_w=bw, block_h=bh, **kw)


def test_block_1x1_is_the_plain_cost():
    """block 1 x 1 = plain SGM, so CB == C and SGM on it is unchanged."""
    rng = np.random.default_rng(5)
    p = _p(9, 7, 5, 1, 1, paths=8)
    C = rng.integers(0, 5, size=(7, 9, 5)).astype(np.uint8)
    CB = oracle.block_cost(p, C)
    assert np.array_equal(CB, C.astype(np.uint32))
    assert np.array_equal(oracle.sgm32(p, CB), oracle.sgm(p, C))


@pytest.mark.parametrize("bw,bh", [(3, 3), (5, 3), (1, 5), (7, 7)])
def test_uniform_cost_one(bw, bh):
    """a 3x3 block on uniform cost 1 gives 9 in the interior; near the
    border each off-image block position contributes nb instead (closed form)."""
    W, H, D = 11, 9, 2
    p = _p(W, H, D, bw, bh)
    nb = p.nbits
    CB = oracle.block_cost(p, np.ones((H, W, D), np.uint8))
    bu, bv = bw // 2, bh // 2
    for y in range(H):
        for x in range(W):
            nx = min(x + bu, W - 1) - max(x - bu, 0) + 1
            ny = min(y + bv, H - 1) - max(y - bv, 0) + 1
            n_in = nx * ny
            expect = n_in + (bw * bh - n_in) * nb
            assert (CB[y, x] == expect).all(), (x, y)
    assert (CB[bv:H - bv, bu:W - bu] == bw * bh).all()


@pytest.mark.parametrize("bw,bh", [(3, 3), (5, 5), (3, 7)])
def test_matches_padded_box_filter(bw, bh):
    """An independent box filter: pad C with nb, sum the bw*bh shifted copies."""
    rng = np.random.default_rng(bw * 10 + bh)
    W, H, D = 13, 10, 4
    p = _p(W, H, D, bw, bh, cw=5, ch=5)
    C = rng.integers(0, p.nbits + 1, size=(H, W, D)).astype(np.uint8)
    bu, bv = bw // 2, bh // 2
    P = np.pad(C.astype(np.int64), ((bv, bv), (bu, bu), (0, 0)), constant_values=p.nbits)
    ref = sum(P[v:v + H, u:u + W] for v in range(bh) for u in range(bw))
    assert np.array_equal(oracle.block_cost(p, C).astype(np.int64), ref)


@pytest.mark.parametrize("paths", [4, 8])
def test_sgm_on_block_costs_bruteforce(paths):
    """O3 on u32 block-cost volumes (values beyond u8) equals exhaustive DP."""
    rng = np.random.default_rng(77 + paths)
    for _ in range(200):
        W, H, D = rng.integers(1, 6), rng.integers(1, 6), rng.integers(1, 5)
        p1 = int(rng.integers(0, 80))
        p2 = int(rng.integers(p1, 300))
        C = rng.integers(0, 400, size=(H, W, D)).astype(np.uint32)
        p = _p(W, H, D, 3, 3, p1=p1, p2=p2, paths=paths)
        S = oracle.sgm32(p, C)
        assert np.array_equal(S.astype(np.int64), aggregate_bruteforce(C.astype(np.int64), p1, p2, paths))


def test_sgbm_recovers_integer_shift():
    """SGBM on the config-A random-dot pair shifted +7 (SimSense supports
    SGBM): >= 99% of the interior (census + block margins) has d* = 7.
    Penalties scale with the block area (P1 = 8*area, P2 = 32*area)."""
    left, right, _ = synth.shift_pair(64, 48, 7, frame_idx=0)
    d = synth.CONFIGS["A"].params_dict()
    d.update(block_w=3, block_h=3, p1=8 * 9, p2=32 * 9)
    p = oracle.Params(**d)
    o = oracle.compute(p, left, right)
    R, Q = p.census_w // 2 + 1, p.census_h // 2 + 1
    inner = o["dstar_l"][Q:p.height - Q, R + 7:p.width - R]
    assert (inner == 7).mean() >= 0.99


def test_sampled_pixel_route_matches_full_volume():
    """oracle_sgm_pixel_from_census restates the block cost per line pixel; it
    must agree with block_cost + sgm32 on the whole image."""
    left, right, _ = synth.shift_pair(40, 30, 3, frame_idx=1)
    d = synth.CONFIGS["A"].params_dict()
    d.update(width=40, height=30, block_w=3, block_h=5, p1=40, p2=150, paths=8)
    p = oracle.Params(**d)
    o = oracle.compute(p, left, right, debug=True)
    for (x, y) in [(0, 0), (39, 29), (17, 11), (5, 28), (33, 2)]:
        s = oracle.sgm_pixel(p, o["census_l"], o["census_r"], x, y)
        assert np.array_equal(s, o["agg"][y, x])

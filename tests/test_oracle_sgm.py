"""Pins for oracle O3 (SGM path aggregation)."""
import json
import os

import numpy as np
import pytest

import oracle
from tests.brute_sgm import aggregate_bruteforce, line_costs_bruteforce

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _params(W, H, D, p1, p2, paths):
    return oracle.Params(width=W, height=H, num_disp=D, census_w=3, census_h=3,
                         p1=p1, p2=p2, paths=paths)


def test_golden_chain_s313():
    """SPEC S:313 hand-sized chain (N=4, D=3, P1=1, P2=2)."""
    g = json.load(open(os.path.join(GOLD, "sgm_chain_n4_d3.json")))
    C = np.array(g["cost"], np.uint32)
    fwd = oracle.chain(C, g["p1"], g["p2"])
    bwd = oracle.chain(C[::-1], g["p1"], g["p2"])[::-1]
    assert fwd.tolist() == g["L_forward"]
    assert bwd.tolist() == g["L_backward"]
    assert (fwd + bwd).tolist() == g["S"]
    assert np.argmin(fwd + bwd, axis=1).tolist() == g["dstar"]
    # and the fixture itself agrees with exhaustive enumeration
    assert line_costs_bruteforce(C.astype(np.int64), g["p1"], g["p2"]).tolist() == g["L_forward"]
    # the 2-D sgm (4-path) on a 1-row image: vertical paths contribute C each
    p = _params(4, 1, 3, g["p1"], g["p2"], 4)
    S = oracle.sgm(p, C.astype(np.uint8)[None])
    assert (S[0] - 2 * C).tolist() == g["S"]


@pytest.mark.parametrize("paths", [4, 8])
def test_bruteforce_random_volumes(paths):
    """SPEC S:376 / acceptance #3: random volumes <= 6x6x4 equal exhaustive DP, exactly."""
    rng = np.random.default_rng(1234 + paths)
    for _ in range(1000):
        W, H, D = rng.integers(1, 7), rng.integers(1, 7), rng.integers(1, 5)
        p1 = int(rng.integers(0, 6))
        p2 = int(rng.integers(p1, 12))
        C = rng.integers(0, 10, size=(H, W, D)).astype(np.uint8)
        S = oracle.sgm(_params(W, H, D, p1, p2, paths), C)
        assert np.array_equal(S.astype(np.int64), aggregate_bruteforce(C, p1, p2, paths))


@pytest.mark.parametrize("paths", [4, 8])
def test_bruteforce_full_6x6x4(paths):
    rng = np.random.default_rng(99 + paths)
    for _ in range(8):
        C = rng.integers(0, 32, size=(6, 6, 4)).astype(np.uint8)
        S = oracle.sgm(_params(6, 6, 4, 8, 32, paths), C)
        assert np.array_equal(S.astype(np.int64), aggregate_bruteforce(C, 8, 32, paths))
        S2 = oracle.sgm(_params(6, 6, 4, 3, 5, paths), C)
        assert np.array_equal(S2.astype(np.int64), aggregate_bruteforce(C, 3, 5, paths))


@pytest.mark.parametrize("paths", [4, 8])
def test_zero_penalties_reduce_to_raw_cost(paths):
    """P1=P2=0 -> S = paths * C, so the argmin is the raw-cost argmin."""
    rng = np.random.default_rng(7)
    C = rng.integers(0, 31, size=(13, 17, 16)).astype(np.uint8)
    S = oracle.sgm(_params(17, 13, 16, 0, 0, paths), C)
    assert np.array_equal(S, paths * C.astype(np.uint32))


@pytest.mark.parametrize("paths", [4, 8])
def test_constant_volume_and_bounds(paths):
    """constant volume -> S constant per pixel; C <= L_r <= C + P2."""
    C = np.full((9, 11, 8), 5, np.uint8)
    S = oracle.sgm(_params(11, 9, 8, 8, 32, paths), C)
    assert (S == S[:, :, :1]).all()
    rng = np.random.default_rng(3)
    C = rng.integers(0, 31, size=(9, 11, 8)).astype(np.uint8)
    p = _params(11, 9, 8, 8, 32, paths)
    for (rx, ry) in oracle.directions(paths):
        L = oracle.sgm_path(p, C, rx, ry).astype(np.int64)
        assert (L >= C).all() and (L <= C.astype(np.int64) + 32).all()


def test_pixel_walk_matches_full_volume():
    """oracle_sgm_pixel_from_census (used at full size) == the full-volume oracle."""
    rng = np.random.default_rng(11)
    p = oracle.Params(width=40, height=30, num_disp=16, census_w=5, census_h=5, paths=8)
    L = rng.integers(0, 256, size=(30, 40), dtype=np.uint8)
    R = rng.integers(0, 256, size=(30, 40), dtype=np.uint8)
    cl, cr = oracle.census(p, L), oracle.census(p, R)
    S = oracle.sgm(p, oracle.cost(p, cl, cr))
    for (x, y) in [(0, 0), (39, 29), (17, 3), (5, 28), (20, 15)]:
        assert np.array_equal(oracle.sgm_pixel(p, cl, cr, x, y), S[y, x])

"""Pins for the R2 right view (oracle O6b; "run the pipeline with
roles swapped", reading c24)."""
import numpy as np
import pytest

import oracle
import synth


def _popcount(a):
    a = a.astype(np.uint64)
    return np.array([bin(int(v)).count("1") for v in a.ravel()]).reshape(a.shape)


def test_cost_right_definition():
    """C_R(x,y,d) = popc(cr(x) ^ cl(x + delta)), nb when x + delta >= W or a
    census window is invalid -- restated in numpy from the census arrays."""
    rng = np.random.default_rng(0)
    W, H, D, mind = 17, 9, 5, 2
    p = oracle.Params(width=W, height=H, num_disp=D, min_disp=mind, census_w=3, census_h=3)
    L = rng.integers(0, 256, (H, W)).astype(np.uint8)
    R = rng.integers(0, 256, (H, W)).astype(np.uint8)
    cl, cr = oracle.census(p, L), oracle.census(p, R)
    CR = oracle.cost_right(p, cl, cr)
    nb = p.nbits
    for y in range(H):
        for x in range(W):
            for d in range(D):
                xl = x + mind + d
                ok = 1 <= y < H - 1 and 1 <= x < W - 1 and xl < W - 1
                want = _popcount(np.uint64(cr[y, x]) ^ np.uint64(cl[y, xl])) if ok else nb
                assert CR[y, x, d] == want, (x, y, d)


def _tie_free_pair(W, H, seed):
    """Rows that are permutations of distinct values: no ties between the two
    pixels of any centre-row census pair."""
    rng = np.random.default_rng(seed)
    L = np.stack([rng.permutation(256)[:W] for _ in range(H)]).astype(np.uint8)
    R = np.stack([rng.permutation(256)[:W] for _ in range(H)]).astype(np.uint8)
    return L, R


@pytest.mark.parametrize("paths,mind", [(4, 0), (8, 0), (8, 3)])
def test_r2_is_the_mirrored_left_view(paths, mind):
    """Matching right-against-left equals matching the mirrored pair with the
    mirrored right image as reference: R2's right view of (L, R) == the flipped
    left view of (flip R, flip L).  Exact when no centre-row census pair ties
    (mirroring maps every other pair to a pair of the same window)."""
    W, H = 48, 20
    L, R = _tie_free_pair(W, H, paths + mind)
    kw = dict(width=W, height=H, num_disp=16, min_disp=mind, census_w=5, census_h=5, paths=paths)
    o = oracle.compute(oracle.Params(**kw, lr_mode=1), L, R)
    m = oracle.compute(oracle.Params(**kw), np.ascontiguousarray(R[:, ::-1]), np.ascontiguousarray(L[:, ::-1]))
    assert np.array_equal(o["dstar_r"], m["dstar_l"][:, ::-1])
    assert np.array_equal(o["dr"].view(np.uint32), m["dl"][:, ::-1].view(np.uint32))
    assert np.array_equal(o["mask_r"] & 3, m["mask"][:, ::-1] & 3)


def test_r2_shift_recovered_and_lr():
    left, right, _ = synth.shift_pair(64, 48, 7, frame_idx=0)
    d = synth.CONFIGS["A"].params_dict()
    o = oracle.compute(oracle.Params(**d, lr_mode=1), left, right)
    R_, Q = 2, 2
    assert (o["dstar_r"][Q:-Q, R_:64 - R_ - 7] == 7).mean() >= 0.99
    inner = np.zeros((48, 64), bool)
    inner[Q:-Q, R_ + 7:64 - R_] = True
    assert ((o["mask"][inner] & oracle.MASK_LR) != 0).mean() <= 0.01

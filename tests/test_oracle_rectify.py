"""Pins for oracle O00 (rectification, reading c23)."""
import numpy as np
import pytest
from scipy import ndimage

import oracle


def _img(H=40, W=56, seed=0):
    return np.random.default_rng(seed).integers(0, 256, (H, W)).astype(np.uint8)


def test_identity_is_bit_identical():
    """identity homographies -> output bit-identical to input."""
    img = _img()
    assert np.array_equal(oracle.rectify(np.eye(3), img), img)


def test_pure_x_shift():
    """a pure x-shift homography by +3 px -> the input translated 3 px
    (out(x) = in(x + 3); the last 3 columns sample outside the image -> 0)."""
    img = _img()
    Hm = np.array([[1, 0, 3], [0, 1, 0], [0, 0, 1]], float)
    out = oracle.rectify(Hm, img)
    assert np.array_equal(out[:, :-3], img[:, 3:])
    assert (out[:, -3:] == 0).all()


def test_singular_rejected():
    """a non-invertible matrix is an error."""
    with pytest.raises(ValueError):
        oracle.rectify(np.array([[1, 2, 0], [2, 4, 0], [0, 0, 1]], float), _img())


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_matches_scipy_bilinear(seed):
    """An independent bilinear resampler (scipy.ndimage.map_coordinates, order 1,
    mode grid-constant = the image zero-padded, as reading c23),
    zero outside) on a random small rotation + perspective: same u8 everywhere
    except where the interpolated value sits within 1e-9 of a rounding tie."""
    rng = np.random.default_rng(seed)
    img = _img(seed=seed).astype(np.float64)
    H, W = img.shape
    ang = rng.uniform(-0.05, 0.05)
    Hm = np.array([[np.cos(ang), -np.sin(ang), rng.uniform(-2, 2)],
                   [np.sin(ang), np.cos(ang), rng.uniform(-2, 2)],
                   [rng.uniform(-1e-4, 1e-4), rng.uniform(-1e-4, 1e-4), 1.0]])
    out = oracle.rectify(Hm, img.astype(np.uint8))
    ys, xs = np.mgrid[0:H, 0:W].astype(np.float64)
    w = Hm[2, 0] * xs + Hm[2, 1] * ys + Hm[2, 2]
    u = (Hm[0, 0] * xs + Hm[0, 1] * ys + Hm[0, 2]) / w
    v = (Hm[1, 0] * xs + Hm[1, 1] * ys + Hm[1, 2]) / w
    ref = ndimage.map_coordinates(img, [v, u], order=1, mode="grid-constant", cval=0.0)
    refq = np.clip(np.floor(ref + 0.5), 0, 255)
    tie = np.abs((ref + 0.5) - np.round(ref + 0.5)) < 1e-9
    assert (out[~tie] == refq[~tie]).all()

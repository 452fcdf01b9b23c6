"""Sensor noise front end on the GPU vs the oracle (
PAPER.md P:275-281; readings c17, c22): same Philox streams, same
Marsaglia-Tsang / Box-Muller steps, fp64 on both sides -> identical u8."""
import numpy as np
import pytest

import oracle
import paper_2201_11924_b200 as asd
import synth
from tests.gpu_util import compare_full, gpu_debug

pytestmark = pytest.mark.gpu


def _both(clean, seed, frame0=0, view=0, **noise):
    import torch
    g = asd.sensor_noise(torch.from_numpy(np.ascontiguousarray(clean, np.float32)).cuda(), seed,
                         frame0=frame0, view=view, **noise)
    torch.cuda.synchronize()
    o = oracle.sensor_noise(np.asarray(clean, np.float32).astype(np.float64), seed, frame0=frame0,
                            view=view, **noise)
    return g.cpu().numpy(), o


@pytest.mark.parametrize("noise", [{}, {"k": 0.6, "theta": 1.4}, {"scale": 0.5}, {"scale": 0.0},
                                   {"sigma": 0.0, "mu": 2.0}])
def test_noise_matches_oracle(noise):
    rng = np.random.default_rng(3)
    clean = rng.uniform(0, 260, (3, 61, 97)).astype(np.float32)
    clean[:, :4] = 0.0
    for view in (0, 1):
        g, o = _both(clean, seed=0x1234_5678_9ABC, frame0=17, view=view, **noise)
        assert np.array_equal(g, o), (np.argwhere(g != o)[:5], (g != o).sum())


def test_noise_frame_offsets_and_seed():
    clean = np.full((2, 40, 50), 120.0, np.float32)
    g0, _ = _both(clean, seed=9)
    g1, _ = _both(clean[:1], seed=9, frame0=1)
    assert np.array_equal(g0[1], g1[0])
    g2, _ = _both(clean, seed=10)
    assert not np.array_equal(g0, g2)


def test_noisy_pair_through_the_depth_path():
    """Datagen order: clean IR pair -> noise -> census/SGM/... ; the
    GPU-noised pair equals the oracle-noised pair and the depth path stays
    bit-exact on it (config A shift scene)."""
    import torch
    cfg = synth.CONFIGS["A"]
    _, _, _ = synth.shift_pair(64, 48, 7, frame_idx=0)
    rng = np.random.default_rng(5)
    T = rng.uniform(20, 200, (48, 80)).astype(np.float32)
    left_c = T[:, :64].copy()
    right_c = T[:, 7:71].copy()                          # right(x) = T(x + 7), reading c5
    gl, ol = _both(left_c, seed=77, view=0)
    gr, orr = _both(right_c, seed=77, view=1)
    assert np.array_equal(gl, ol) and np.array_equal(gr, orr)
    d = cfg.params_dict()
    g = gpu_debug(d, gl, gr)
    o = oracle.compute(oracle.Params(**d), ol, orr, debug=True)
    compare_full(g, o)

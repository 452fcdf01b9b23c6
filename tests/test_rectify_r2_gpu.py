"""Rectification and the R2 right view on the GPU vs the oracle (SURVEY §8(f)
NEXT 4; readings c23, c24)."""
import numpy as np
import pytest

import oracle
import paper_2201_11924_b200 as asd
import synth
from tests.gpu_util import compare_full, gpu_debug

pytestmark = pytest.mark.gpu


def _rect_both(Hm, imgs):
    import torch
    g = asd.rectify(Hm, torch.from_numpy(np.ascontiguousarray(imgs)).cuda())
    torch.cuda.synchronize()
    g = g.cpu().numpy()
    for i in range(imgs.shape[0]):
        assert np.array_equal(g[i], oracle.rectify(Hm, imgs[i])), f"image {i}"
    return g


def test_rectify_identity_shift_and_random():
    rng = np.random.default_rng(4)
    imgs = rng.integers(0, 256, (3, 45, 70)).astype(np.uint8)
    g = _rect_both(np.eye(3), imgs)
    assert np.array_equal(g, imgs)
    g = _rect_both(np.array([[1, 0, 3], [0, 1, 0], [0, 0, 1]], float), imgs)
    assert np.array_equal(g[:, :, :-3], imgs[:, :, 3:])
    for seed in range(3):
        r = np.random.default_rng(seed)
        a = r.uniform(-0.04, 0.04)
        Hm = np.array([[np.cos(a), -np.sin(a), r.uniform(-3, 3)], [np.sin(a), np.cos(a), r.uniform(-3, 3)],
                       [r.uniform(-2e-4, 2e-4), r.uniform(-2e-4, 2e-4), 1.0]])
        _rect_both(Hm, imgs)


def test_rectified_pair_through_the_depth_path():
    """A pair misaligned by a small vertical offset and rotation, rectified with
    the inverse homographies, then matched: every stage bit-exact."""
    import torch
    left, right, _ = synth.shift_pair(64, 48, 7, frame_idx=1)
    Hr = np.array([[1, 0, 0], [0, 1, 0.5], [0, 0, 1]], float)
    rl = _rect_both(np.eye(3), left[None])[0]
    rr = _rect_both(Hr, right[None])[0]
    d = synth.CONFIGS["A"].params_dict()
    compare_full(gpu_debug(d, rl, rr), oracle.compute(oracle.Params(**d), rl, rr, debug=True))


@pytest.mark.parametrize("paths,mind,block,median,engine", [
    (4, 0, 1, 0, 1), (8, 0, 1, 0, 1), (8, 2, 1, 0, 1), (8, 0, 3, 0, 1), (8, 0, 1, 3, 1),
    (4, 0, 1, 0, 3), (8, 0, 1, 0, 3), (8, 2, 1, 0, 3), (8, 0, 1, 3, 3)])
def test_r2_config_A(paths, mind, block, median, engine):
    left, right, _ = synth.shift_pair(64, 48, 7, frame_idx=2)
    d = dict(synth.CONFIGS["A"].params_dict(), paths=paths, min_disp=mind, lr_mode=1,
             median_ksize=median)
    if block > 1:
        d.update(block_w=block, block_h=block, p1=8 * block * block, p2=32 * block * block)
    g = gpu_debug(d, left, right, engine=engine)
    o = oracle.compute(oracle.Params(**d), left, right, debug=True)
    compare_full(g, o)


@pytest.mark.parametrize("engine", [1, 3])
def test_r2_config_B_full_frame(engine):
    cfg = synth.CONFIGS["B"]
    left, right = synth.make_pair(cfg, 3)[:2]
    d = dict(cfg.params_dict(), lr_mode=1)
    compare_full(gpu_debug(d, left, right, engine=engine),
                 oracle.compute(oracle.Params(**d), left, right, debug=True))


def test_r2_d3_batch_config_C():
    """R2 inside the D3 group pipeline at config C (3 frames, groups of 2):
    per-frame outputs and checksums equal the oracle's."""
    import torch
    from tests.gpu_util import assert_bits_equal, assert_depth_close
    cfg = synth.CONFIGS["C"]
    d = dict(cfg.params_dict(), lr_mode=1)
    Ls, Rs = synth.frame_pool(cfg, 3)
    with asd.Stereo(asd.Params(**d), 0, 4) as st:
        assert st.engine == 3
        st.group = 2
        L = torch.from_numpy(Ls).cuda(); R = torch.from_numpy(Rs).cuda()
        disp = torch.empty(3, cfg.height, cfg.width, device="cuda")
        depth = torch.empty_like(disp)
        stats = torch.zeros(3, 4, dtype=torch.int32, device="cuda")
        st.asd_depth_batch(L, R, disp, depth, stats)
        torch.cuda.synchronize()
    disp, depth, stats = disp.cpu().numpy(), depth.cpu().numpy(), stats.cpu().numpy()
    op = oracle.Params(**d)
    for i in range(3):
        o = oracle.compute(op, Ls[i], Rs[i])
        assert_bits_equal(disp[i], o["disp"], f"disp {i}")
        assert_depth_close(depth[i], o["depth"])
        assert int(stats[i, 0]) & 0xFFFFFFFF == oracle.checksum(o["dstar_l"], o["mask"])

"""Median filter and depth registration on the GPU vs the oracle (SURVEY §8(f)
NEXT 2; readings c20, c21).
Both are bit-exact: the median compares fp32 values, the registration's fp32
coordinate arithmetic is the same sequence of IEEE operations on both sides."""
import numpy as np
import pytest

import oracle
import paper_2201_11924_b200 as asd
import synth
from tests.gpu_util import assert_bits_equal, assert_depth_close, compare_full, gpu_debug

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k,engine", [(3, 0), (5, 0), (3, 1), (5, 1)])
def test_median_config_A(k, engine):
    left, right, _ = synth.shift_pair(64, 48, 7, frame_idx=1)
    d = dict(synth.CONFIGS["A"].params_dict(), median_ksize=k)
    g = gpu_debug(d, left, right, engine=engine)
    o = oracle.compute(oracle.Params(**d), left, right, debug=True)
    compare_full(g, o)


@pytest.mark.parametrize("k", [3, 5])
def test_median_config_B_full_frame(k):
    cfg = synth.CONFIGS["B"]
    left, right = synth.make_pair(cfg, 2)[:2]
    d = dict(cfg.params_dict(), median_ksize=k)
    g = gpu_debug(d, left, right)
    o = oracle.compute(oracle.Params(**d), left, right, debug=True)
    compare_full(g, o)


def test_median_batch_pipeline():
    """Median inside the D3 group pipeline (config B, 5 frames, groups of 2)."""
    import torch
    cfg = synth.CONFIGS["B"]
    d = dict(cfg.params_dict(), median_ksize=5)
    Ls, Rs = synth.frame_pool(cfg, 5)
    with asd.Stereo(asd.Params(**d), 0, 4) as st:
        if st.engine == 3:
            st.group = 2
        L = torch.from_numpy(Ls).cuda(); R = torch.from_numpy(Rs).cuda()
        disp = torch.empty(5, cfg.height, cfg.width, device="cuda")
        depth = torch.empty_like(disp)
        stats = torch.zeros(5, 4, dtype=torch.int32, device="cuda")
        st.asd_depth_batch(L, R, disp, depth, stats)
        torch.cuda.synchronize()
    disp, depth, stats = disp.cpu().numpy(), depth.cpu().numpy(), stats.cpu().numpy()
    op = oracle.Params(**d)
    for i in range(5):
        o = oracle.compute(op, Ls[i], Rs[i])
        assert_bits_equal(disp[i], o["disp"], f"disp {i}")
        assert_depth_close(depth[i], o["depth"])
        assert int(stats[i, 0]) & 0xFFFFFFFF == oracle.checksum(o["dstar_l"], o["mask"])


CAM = (40, 30, 100.0, 100.0, 19.5, 14.5)
EYE = np.eye(3, dtype=np.float32)


def _reg_both(ir, rgb, R, t, z):
    import torch
    g = asd.register_depth(ir, rgb, R, t, torch.from_numpy(np.ascontiguousarray(z)).cuda())
    torch.cuda.synchronize()
    g = g.cpu().numpy()
    zs = z if z.ndim == 3 else z[None]
    gs = g if g.ndim == 3 else g[None]
    for i in range(zs.shape[0]):
        o = oracle.register(ir, rgb, R, t, zs[i])
        assert_bits_equal(gs[i], o, f"registered frame {i}")
    return g


def test_register_identity_and_translation():
    rng = np.random.default_rng(3)
    z = rng.uniform(0.3, 3.0, (30, 40)).astype(np.float32)
    z[rng.random((30, 40)) < 0.2] = np.nan
    g = _reg_both(CAM, CAM, EYE, [0, 0, 0], z)
    assert np.array_equal(np.isnan(g), np.isnan(z))
    wall = np.ones((30, 40), np.float32)
    g = _reg_both(CAM, CAM, EYE, [-0.05, 0, 0], wall)
    assert (g[:, :35] == 1.0).all() and np.isnan(g[:, 35:]).all()


def test_register_random_rigid_batch():
    """Random depth maps, a rotation + translation, a larger RGB camera, 3 frames."""
    rng = np.random.default_rng(11)
    ir = (64, 48, 120.0, 121.0, 31.5, 23.5)
    rgb = (96, 72, 180.0, 181.0, 47.0, 35.0)
    ang = 0.05
    R = np.array([[np.cos(ang), 0, np.sin(ang)], [0, 1, 0], [-np.sin(ang), 0, np.cos(ang)]], np.float32)
    z = rng.uniform(0.4, 2.0, (3, 48, 64)).astype(np.float32)
    z[rng.random((3, 48, 64)) < 0.1] = np.nan
    z[1, :5] = 0.0
    z[2, 10:20] = -1.0
    _reg_both(ir, rgb, R, [-0.015, 0.002, 0.001], z)


def test_register_pipeline_depth_to_rgb_1080p():
    """Config B depth (asd_depth) registered to a 1920x1080 RGB camera (the
    Table II output resolution, reading c16) with a D415-like 15 mm offset."""
    import torch
    cfg = synth.CONFIGS["B"]
    left, right = synth.make_pair(cfg, 0)[:2]
    with asd.Stereo(asd.Params(**cfg.params_dict()), 0, 1) as st:
        L = torch.from_numpy(left).cuda(); Rr = torch.from_numpy(right).cuda()
        disp = torch.empty(cfg.height, cfg.width, device="cuda")
        depth = torch.empty_like(disp)
        st.asd_depth(L, Rr, disp, depth)
        torch.cuda.synchronize()
    z = depth.cpu().numpy()
    ir = (cfg.width, cfg.height, cfg.focal_px, cfg.focal_px, (cfg.width - 1) / 2, (cfg.height - 1) / 2)
    f_rgb = 1380.0
    rgb = (1920, 1080, f_rgb, f_rgb, 959.5, 539.5)
    g = _reg_both(ir, rgb, EYE, [-0.015, 0.0, 0.0], z)
    assert (~np.isnan(g)).sum() > 0.5 * (~np.isnan(z)).sum()


def test_register_empty_batch():
    import torch
    out = torch.empty(0, 30, 40, device="cuda")
    r = asd.register_depth(CAM, CAM, EYE, [0, 0, 0], torch.empty(0, 30, 40, device="cuda"), out)
    assert r.shape == (0, 30, 40)

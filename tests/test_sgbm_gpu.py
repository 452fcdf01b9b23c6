"""SGBM (reading c19) on the
GPU vs the oracle: block cost volume -> D1 aggregation -> WTA/LR/depth, every
stage output bit-exact (depth within 1e-5)."""
import numpy as np
import pytest

import oracle
import paper_2201_11924_b200 as asd
import synth
from tests.gpu_util import compare_full, gpu_debug, assert_bits_equal, assert_depth_close

pytestmark = pytest.mark.gpu


def _cfg(name, bw, bh, paths=None, **kw):
    d = synth.CONFIGS[name].params_dict()
    d.update(block_w=bw, block_h=bh, p1=8 * bw * bh, p2=32 * bw * bh)
    if paths:
        d["paths"] = paths
    d.update(kw)
    return d


@pytest.mark.parametrize("bw,bh,paths", [(3, 3, 4), (3, 3, 8), (5, 3, 8), (1, 5, 8), (7, 7, 4)])
def test_sgbm_config_A_all_stages(bw, bh, paths):
    left, right, _ = synth.shift_pair(64, 48, 7, frame_idx=2)
    d = _cfg("A", bw, bh, paths)
    g = gpu_debug(d, left, right)
    o = oracle.compute(oracle.Params(**d), left, right, debug=True)
    compare_full(g, o)


def test_sgbm_fractional_shift_and_minimum_disparity():
    """A non-integer shift with min_disp > 0 and a ragged width (not a multiple
    of the 32-pixel CTA tile)."""
    left, right, _ = synth.shift_pair(77, 41, 6.5, frame_idx=3)
    d = _cfg("A", 3, 3, 8, width=77, height=41, min_disp=2)
    g = gpu_debug(d, left, right)
    o = oracle.compute(oracle.Params(**d), left, right, debug=True)
    compare_full(g, o)


def test_sgbm_config_B_full_frame():
    """Config B (640x360, D=64, 7x7 census) with a 3x3 block, 8 paths."""
    cfg = synth.CONFIGS["B"]
    left, right = synth.make_pair(cfg, 0)[:2]
    d = _cfg("B", 3, 3)
    g = gpu_debug(d, left, right)
    o = oracle.compute(oracle.Params(**d), left, right, debug=True)
    compare_full(g, o)


def test_sgbm_block_1x1_equals_sgm():
    """block 1 x 1 is plain SGM: same outputs as the default (D3) engine."""
    cfg = synth.CONFIGS["B"]
    left, right = synth.make_pair(cfg, 1)[:2]
    d = cfg.params_dict()
    g0 = gpu_debug(d, left, right)
    g1 = gpu_debug(dict(d, block_w=1, block_h=1), left, right)
    for k in ("dstar_l", "dstar_r", "mask", "mask_r"):
        assert np.array_equal(g0[k], g1[k]), k
    assert_bits_equal(g0["disp"], g1["disp"], "disp")


def test_sgbm_d3_needs_d128():
    """SGBM on engine D3 is built for num_disp = 128 (config A has 16): D1 only."""
    p = asd.Params(**_cfg("A", 3, 3), engine=3)
    with pytest.raises(asd.AsdError) as e:
        asd.Stereo(p, 0, 1)
    assert e.value.code == asd.ASD_E_UNSUPPORTED


@pytest.mark.parametrize("engine", [1, 3])
def test_sgbm_batch_config_C_sampled(engine):
    """Config C with a 3x3 block in a batch of 2 (bench-sized frames) on both
    engines (D3: block cost in the sweeps' private layout, u16 partials): the
    per-frame disparities, depths, checksums and valid counts equal the oracle's."""
    import torch
    cfg = synth.CONFIGS["C"]
    d = _cfg("C", 3, 3)
    Ls, Rs = synth.frame_pool(cfg, 2)
    p = asd.Params(**d, engine=engine)
    with asd.Stereo(p, 0, 2) as st:
        assert st.engine == engine
        L = torch.from_numpy(Ls).cuda(); R = torch.from_numpy(Rs).cuda()
        disp = torch.empty(2, cfg.height, cfg.width, device="cuda")
        depth = torch.empty_like(disp)
        stats = torch.zeros(2, 4, dtype=torch.int32, device="cuda")
        st.asd_depth_batch(L, R, disp, depth, stats)
        torch.cuda.synchronize()
        stats = stats.cpu().numpy()
        disp = disp.cpu().numpy()
        depth = depth.cpu().numpy()
    op = oracle.Params(**d)
    for i in range(2):
        o = oracle.compute(op, Ls[i], Rs[i])
        assert int(stats[i, 0]) & 0xFFFFFFFF == oracle.checksum(o["dstar_l"], o["mask"])
        assert stats[i, 1] == int((o["mask"] == 0).sum())
        assert_bits_equal(disp[i], o["disp"], f"disp frame {i}")
        assert_depth_close(depth[i], o["depth"])

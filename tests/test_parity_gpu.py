"""CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar (BASELINE.json north_star): census, cost, aggregated cost,
integer disparities (left and right), masks, and the float sub-pixel
disparities are bit-exact; depth within 1e-5 relative (fp32 vs fp64)."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import (assert_bits_equal, assert_depth_close, assert_equal, compare_full,
                            gpu_debug)

pytestmark = pytest.mark.gpu

ENGINES = [pytest.param(1, id="D1"), pytest.param(3, id="D3")]


def _cfg(name, **kw):
    d = synth.CONFIGS[name].params_dict()
    d.update(kw)
    return d


def _run(d, left, right, engine=0):
    o = oracle.compute(oracle.Params(**d), left, right, debug=True)
    g = gpu_debug(d, left, right, engine)
    compare_full(g, o)
    return g, o


@pytest.mark.parametrize("engine", ENGINES)
def test_config_A_shift7(engine):
    left, right, _ = synth.make_pair("A", 0)
    g, o = _run(_cfg("A"), left, right, engine)
    assert (g["dstar_l"][2:-2, 9:-2] == 7).mean() >= 0.99


@pytest.mark.parametrize("engine", ENGINES)
def test_config_A_fractional(engine):
    left, right, _ = synth.shift_pair(64, 48, 6.5, frame_idx=3)
    _run(_cfg("A"), left, right, engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_config_B_full(engine):
    left, right, _ = synth.make_pair("B", 0)
    _run(_cfg("B"), left, right, engine)


FUZZ = [
    # W, H, D, min_disp, cw, ch, p1, p2, paths, uniq, lr, subpix
    (37, 23, 16, 0, 5, 5, 8, 32, 4, 10, 1.0, 1),
    (61, 29, 48, 3, 3, 3, 5, 9, 8, 0, 0.5, 1),
    (100, 40, 32, 0, 7, 5, 0, 0, 8, 10, 1.0, 1),
    (129, 17, 64, 17, 9, 7, 8, 32, 8, 25, 2.0, 0),
    (70, 45, 80, 0, 11, 11, 8, 32, 8, 10, 1.0, 1),       # nb = 60 -> u64 census
    (90, 33, 16, 40, 9, 9, 12, 100, 4, -1, -1.0, 1),      # nb = 40 -> u64, no uniq / LR
    (48, 31, 256, 0, 5, 3, 3, 30, 8, 5, 3.0, 1),           # D > W
    (200, 9, 128, 2, 9, 7, 8, 32, 8, 10, 1.0, 1),
    (33, 64, 112, 0, 3, 5, 1, 2, 4, 100, 0.0, 1),
    (16, 16, 16, 0, 15, 1, 200, 248, 8, 10, 1.0, 1),      # nb = 7, p2 near the u8 bound
    (160, 40, 64, 8, 7, 7, 8, 32, 8, 10, 1.0, 1),          # TMA census staging with min_disp > 0
    (264, 24, 128, 12, 9, 7, 8, 32, 8, 10, 1.0, 1),        # the same at D = 128, two CTAs
    (96, 20, 96, 4, 9, 7, 10, 50, 8, 15, 1.5, 1),          # D = 96, P2 = 50 (u32 keys)
    (300, 20, 256, 20, 5, 5, 8, 32, 4, 10, 1.0, 1),        # D = 256, 4 paths, min_disp 20
]


# inside the D3 envelope (nb <= 32, D in {16,32,64,128}, u8 partial, 16-bit keys):
# ragged widths, several cluster CTAs, W < D, P1=P2=0, 4-path at D=128, nb = 32
FUZZ_D3 = [
    (300, 37, 128, 0, 9, 7, 8, 32, 8, 10, 1.0, 1),
    (257, 21, 64, 5, 7, 7, 3, 20, 8, 15, 0.5, 1),
    (129, 40, 32, 0, 5, 5, 0, 0, 8, 10, 1.0, 1),
    (97, 33, 16, 2, 3, 3, 1, 2, 4, 0, 2.0, 0),
    (1000, 12, 128, 3, 13, 5, 10, 30, 8, -1, -1.0, 1),
    (640, 30, 128, 0, 9, 7, 8, 32, 4, 10, 1.0, 1),
    (33, 50, 64, 0, 9, 7, 8, 32, 8, 10, 1.0, 1),
    (2000, 8, 128, 0, 9, 7, 8, 32, 8, 10, 1.0, 1),
]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("case", FUZZ + FUZZ_D3)
def test_fuzz(case, engine):
    W, H, D, md, cw, ch, p1, p2, paths, u, lr, sp = case
    d = dict(width=W, height=H, num_disp=D, min_disp=md, census_w=cw, census_h=ch, p1=p1, p2=p2,
             paths=paths, uniqueness=u, lr_max_diff=lr, subpixel=sp, focal_px=321.5, baseline_m=0.05)
    rng = np.random.default_rng(W * 1000 + H)
    shift = int(rng.integers(0, max(1, min(D, W // 3)))) + md
    T = rng.integers(0, 256, size=(H, W + shift + 1), dtype=np.uint8)
    left = T[:, :W].copy()
    right = T[:, shift:shift + W].copy()
    noise = rng.integers(0, 2, size=right.shape, dtype=np.uint8)
    right = np.where(rng.random(right.shape) < 0.1, right ^ noise, right).astype(np.uint8)
    _run(d, left, right, engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_textureless_and_constant(engine):
    d = _cfg("A")
    z = np.zeros((48, 64), np.uint8)
    g, o = _run(d, z, z, engine)
    assert (g["mask"] != 0).mean() >= 0.99
    c = np.full((48, 64), 200, np.uint8)
    _run(d, c, z, engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_config_C_full_frame(engine):
    """One full 1280x720 D128 8-path frame, every stage, bit-exact."""
    left, right, _ = synth.make_pair("C", 0)
    _run(_cfg("C"), left, right, engine)


@pytest.mark.parametrize("engine", ENGINES)
def test_config_D_full_frame(engine):
    """One full 1920x1080 D256 8-path frame (BASELINE.json configs[3]), every
    stage against the full oracle: census, cost, S, d* of both views, masks and
    sub-pixel disparities bit-exact, depth to 1e-5 (about 9 GB of host memory
    and half a minute of oracle time).  On D3 the frame spans two clusters of
    15 CTAs joined through global memory."""
    left, right, _ = synth.make_pair("D", 0)
    _run(_cfg("D"), left, right, engine)


@pytest.mark.parametrize("p2", [40, 54, 60, 120, 224])
def test_d3_envelope_p2(p2):
    """Engine D3 beyond the 16-bit-key / 8-bit-partial envelope (the
    parameters are adjustable): P2 = 40 and 54 need u32 WTA keys (8 (nb + P2)
    << 7 > 0xFFFE); P2 >= 55 makes the 3-path partial exceed 8 bits, so the
    sweeps run their u16-partial instances on the per-pixel cost (a 1 x 1 block
    cost); 224 = the validated maximum (nb + P2 <= 255).  Every stage bit-exact
    at a 320x96 D=128 8-path speckle pair, and on one full config-C frame at
    P2 = 40 and 120."""
    cfg = synth.StereoConfig("P", 320, 96, 128, 9, 7, 8, 430.0 * 320 / 424, tag=11)
    left, right, _ = synth.speckle_pair(cfg, 0)
    d = dict(cfg.params_dict(), p2=p2)
    _run(d, left, right, 3)
    if p2 in (40, 120):
        left, right, _ = synth.make_pair("C", 1)
        _run(_cfg("C", p2=p2), left, right, 3)


@pytest.mark.parametrize("W,H,D,paths", [(320, 96, 96, 8), (320, 96, 96, 4), (512, 96, 256, 8),
                                         (600, 80, 256, 4), (1000, 40, 256, 8),
                                         (1100, 48, 256, 8), (2100, 40, 128, 8),
                                         (2300, 32, 256, 8), (4400, 24, 128, 8)])
def test_d3_more_disparity_ranges(W, H, D, paths):
    """Engine D3 at D = 96 (DC = 24 disparities per thread, T = 4) and D = 256
    (T = 8 threads per column, 8 disparities per lane in the row kernel, the
    warp-per-pixel WTA): Table II's other disparity ranges and
    P:293's adjustable parameters.  An 8-path frame wider than one cluster
    (16 CTAs of 64 columns at D = 256, of 128 at D = 128: the last four cases)
    runs as two or four clusters joined through global memory at the
    boundaries (tagged-word halos; a middle segment both receives from and
    sends to each side).  Every stage bit-exact."""
    cfg = synth.StereoConfig("R", W, H, D, 9, 7, paths, 430.0 * W / 424 * D / 128, tag=12)
    left, right, _ = synth.speckle_pair(cfg, 0)
    _run(cfg.params_dict(), left, right, 3)


@pytest.mark.parametrize("variant", ["sgbm3", "r2", "p2_100", "median5"])
def test_d3_two_segment_variants(variant):
    """The engine's other instances on a frame spanning two clusters (2100 x 40,
    D = 128, 8 paths): SGBM 3x3 and SGM with P2 = 100 (u16-partial BLK sweeps),
    the R2 right view (right-referenced down sweep), median 5.  Bit-exact."""
    cfg = synth.StereoConfig("S2", 2100, 40, 128, 9, 7, 8, 430.0 * 2100 / 424, tag=13)
    left, right, _ = synth.speckle_pair(cfg, 0)
    d = cfg.params_dict()
    d.update({"sgbm3": dict(block_w=3, block_h=3, p1=72, p2=288), "r2": dict(lr_mode=1),
              "p2_100": dict(p2=100), "median5": dict(median_ksize=5)}[variant])
    _run(d, left, right, 3)


@pytest.mark.parametrize("W,D,min_disp", [(2102, 128, 0), (2100, 128, 3), (1102, 256, 6)])
def test_d3_segments_cp_async_census(W, D, min_disp):
    """Frames spanning two clusters whose census rows are staged with 4-byte
    cp.async instead of TMA (width not a multiple of 4, or min_disp not), so
    the segment receive's cp.async groups interleave with the census groups
    of the down sweep.  Every stage bit-exact."""
    cfg = synth.StereoConfig("SC", W, 32, D, 9, 7, 8, 430.0 * W / 424 * D / 128, min_disp=min_disp, tag=14)
    left, right, _ = synth.speckle_pair(cfg, 0)
    _run(cfg.params_dict(), left, right, 3)

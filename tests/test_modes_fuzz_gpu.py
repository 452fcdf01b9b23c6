"""Seeded fuzz over the optional stages (SGBM block, median, R2 right view)
combined with ragged shapes, both engines: every stage output vs the oracle
(SURVEY §8(f) rows on the same bar as §8(a): bit-exact, depth 1e-5)."""
import numpy as np
import pytest

import oracle
from tests.gpu_util import compare_full, gpu_debug

pytestmark = pytest.mark.gpu

# W, H, D, min_disp, cw, ch, paths, block, median, lr_mode
CASES = [
    (37, 23, 16, 0, 5, 5, 4, 3, 0, 0),
    (61, 29, 32, 3, 3, 3, 8, 1, 3, 1),
    (100, 40, 64, 0, 7, 5, 8, 5, 5, 0),
    (129, 17, 64, 11, 9, 7, 8, 1, 5, 1),
    (70, 45, 48, 0, 5, 5, 8, 3, 3, 1),        # D = 48: D1 only
    (257, 21, 128, 5, 7, 7, 8, 1, 3, 1),
    (300, 37, 128, 0, 9, 7, 8, 1, 0, 1),
    (90, 33, 16, 4, 9, 9, 4, 3, 5, 1),        # nb = 40 (u64 census): D1 only
    (33, 50, 64, 0, 9, 7, 8, 7, 0, 0),
    (12, 9, 16, 0, 3, 3, 8, 3, 3, 1),         # tiny image
    # SGBM at D = 128 (engine D3: block cost in the sweeps' private layout)
    (300, 37, 128, 0, 9, 7, 8, 3, 0, 0),
    (257, 21, 128, 5, 7, 7, 8, 3, 3, 1),
    (130, 20, 128, 2, 5, 5, 8, 5, 0, 1),
    (1283, 9, 128, 0, 9, 7, 8, 3, 5, 0),      # several cluster CTAs, ragged last CTA
    (333, 19, 128, 0, 9, 7, 4, 3, 3, 0),      # 4-path SGBM (D3: vertical-only strips)
    (200, 25, 128, 3, 7, 7, 4, 5, 0, 1),      # 4-path SGBM + R2
    (150, 30, 96, 0, 9, 7, 4, 1, 3, 0),       # D = 96 (D1 with the window WTA kernel)
    (97, 20, 96, 5, 5, 5, 8, 3, 0, 0),        # D = 96 SGBM (u32 WTA keys)
    (300, 21, 256, 0, 9, 7, 4, 1, 3, 0),      # D = 256, 4 paths: packed u16 keys in the window WTA
    (140, 17, 256, 7, 7, 5, 8, 1, 0, 0),      # D = 256, 8 paths: u32 keys
    # engine D1 lane layouts (DPL = D / act): partial warps and lines without an all-valid interval
    (120, 19, 80, 9, 7, 7, 8, 1, 0, 1),       # D = 80: 4 per lane, 20 active lanes, R2
    (260, 15, 144, 20, 9, 7, 8, 1, 0, 0),     # D = 144: 8 per lane, 18 active lanes, min_disp 20
    (60, 12, 240, 0, 5, 5, 4, 1, 0, 1),       # D = 240 > W: every matched window range is partial
    (75, 14, 112, 33, 7, 5, 8, 3, 0, 0),      # D = 112 SGBM (cost from CB), min_disp 33
    # round 2: D3 at D = 256 with R2 + median, and SGBM + median + R2 on a frame spanning two clusters
    (200, 20, 256, 0, 9, 7, 8, 1, 3, 1),
    (2100, 9, 128, 0, 9, 7, 8, 3, 5, 1),
]


@pytest.mark.parametrize("engine", [pytest.param(1, id="D1"), pytest.param(3, id="D3")])
@pytest.mark.parametrize("case", CASES)
def test_modes_fuzz(case, engine):
    W, H, D, md, cw, ch, paths, block, median, lrm = case
    d = dict(width=W, height=H, num_disp=D, min_disp=md, census_w=cw, census_h=ch, paths=paths,
             p1=8 * block * block, p2=32 * block * block, block_w=block, block_h=block,
             median_ksize=median, lr_mode=lrm, uniqueness=10, lr_max_diff=1.0, subpixel=1,
             focal_px=321.5, baseline_m=0.05)
    rng = np.random.default_rng(W * 7 + H * 3 + D)
    shift = int(rng.integers(0, max(1, min(D, W // 3)))) + md
    T = rng.integers(0, 256, size=(H, W + shift + 1), dtype=np.uint8)
    left = T[:, :W].copy()
    right = T[:, shift:shift + W].copy()
    g = gpu_debug(d, left, right, engine)       # skips when outside the D3 envelope
    o = oracle.compute(oracle.Params(**d), left, right, debug=True)
    compare_full(g, o)

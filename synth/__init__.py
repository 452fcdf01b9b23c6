"""Seeded synthetic IR stereo pairs (input generator shared by tests, bench and smoke).

This module holds NONE of the stereo method's arithmetic (no census, cost, SGM,
WTA, sub-pixel, LR or depth-from-disparity computation): it only draws images.
Both the CUDA path and the CPU oracle consume what it produces.

Recipe:
  * Seeds: numpy ``PCG64(SeedSequence([220111924, frame_idx, cfg_tag]))``.
  * Config A: i.i.d. uniform u8 random-dot texture T; left(x) = T(x),
    right(x) = T(x + s) for a known shift s.  The
    fractional variant samples T bilinearly at x + 6.5.
  * Configs B/C/D: D415-shaped speckle scenes.  Ground-truth depth in the left
    view: background plane at 1.8 m, a slanted plane 0.7-1.4 m, 3-6 boxes at
    0.6-1.2 m and one "transparent" disk that carries no projector pattern
    (the holes of P:7 / P:29).  The projector sits at the left camera, so the
    left image shows the Bernoulli dot pattern (density 0.25, 180 DN, ~1 px
    blobs) over a 20 DN ambient; the right image is a z-buffered forward warp
    of the left intensity with bilinear sampling, and right pixels that no
    left surface reaches are in the projector's shadow (ambient only).
  * Sensor noise (parameters P:350: k=3.98, theta=0.254,
    mu=-0.231, sigma=0.83, in DN): I = gamma*I_clean + n, then round half up
    and clamp to u8 (reading c17).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 220111924

# Sensor noise parameters estimated for the D415.
NOISE_K, NOISE_THETA, NOISE_MU, NOISE_SIGMA = 3.98, 0.254, -0.231, 0.83


@dataclass(frozen=True)
class StereoConfig:
    """One BASELINE.json config (names A-E follow SURVEY §8(a))."""
    name: str
    width: int
    height: int
    num_disp: int
    census_w: int
    census_h: int
    paths: int
    focal_px: float
    baseline_m: float = 0.055          # D415 baseline
    min_disp: int = 0
    p1: int = 8                        # SPEC defaults S:388 (reading c7)
    p2: int = 32
    uniqueness: int = 10
    lr_max_diff: float = 1.0
    subpixel: int = 1
    frames: int = 1
    kind: str = "speckle"
    tag: int = field(default=0)

    @property
    def cells(self) -> int:
        return self.width * self.height * self.num_disp

    def params_dict(self) -> dict:
        return dict(width=self.width, height=self.height, min_disp=self.min_disp,
                    num_disp=self.num_disp, census_w=self.census_w, census_h=self.census_h,
                    p1=self.p1, p2=self.p2, paths=self.paths, uniqueness=self.uniqueness,
                    lr_max_diff=self.lr_max_diff, subpixel=self.subpixel,
                    focal_px=self.focal_px, baseline_m=self.baseline_m)


def _f(w: int) -> float:
    """SPEC's fx = 430 px at 424x240, scaled with the width."""
    return float(np.float32(430.0 * w / 424.0))


CONFIGS = {
    "A": StereoConfig("A", 64, 48, 16, 5, 5, 4, _f(64), kind="shift", tag=1),
    "B": StereoConfig("B", 640, 360, 64, 7, 7, 8, _f(640), tag=2),
    "C": StereoConfig("C", 1280, 720, 128, 9, 7, 8, _f(1280), tag=3),
    "D": StereoConfig("D", 1920, 1080, 256, 9, 7, 8, _f(1920), tag=4),
    "E": StereoConfig("E", 1280, 720, 128, 9, 7, 8, _f(1280), frames=4096, tag=3),
    # the paper's Table II workload: 960x540 input, 4-path SGM,
    # max disparity 64 / 96 / 128 / 256 (census window unstated: 9x7, as C)
    "T64": StereoConfig("T64", 960, 540, 64, 9, 7, 4, _f(960), tag=5),
    "T96": StereoConfig("T96", 960, 540, 96, 9, 7, 4, _f(960), tag=5),
    "T128": StereoConfig("T128", 960, 540, 128, 9, 7, 4, _f(960), tag=5),
    "T256": StereoConfig("T256", 960, 540, 256, 9, 7, 4, _f(960), tag=5),
}


def rng_for(frame_idx: int, tag: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([SEED_BASE, frame_idx, tag])))


def quantize(img: np.ndarray) -> np.ndarray:
    """Round half up, clamp to [0, 255] (reading c17)."""
    return np.clip(np.floor(img + 0.5), 0, 255).astype(np.uint8)


def apply_noise(clean: np.ndarray, rng: np.random.Generator, scale: float = 1.0) -> np.ndarray:
    """I_noisy = gamma * I_clean + n; gamma ~ Gamma(k, theta), n ~ N(mu, sigma^2)."""
    g = rng.gamma(NOISE_K, NOISE_THETA, size=clean.shape)
    n = rng.normal(NOISE_MU, NOISE_SIGMA, size=clean.shape)
    if scale != 1.0:
        kt = NOISE_K * NOISE_THETA
        g = kt + scale * (g - kt)
        n = scale * n
    return g * clean + n


def shift_pair(width: int, height: int, shift: float, frame_idx: int = 0, tag: int = 1):
    """Random-dot pair with a known horizontal shift.

    left(x) = T(x), right(x) = T(x + shift); T is i.i.d. uniform u8.  A
    fractional shift samples T bilinearly.  Ground truth disparity = shift.
    """
    rng = rng_for(frame_idx, tag)
    extra = int(np.ceil(shift)) + 1
    T = rng.integers(0, 256, size=(height, width + extra), dtype=np.uint8)
    left = T[:, :width].copy()
    s = float(shift)
    i0 = int(np.floor(s))
    t = s - i0
    if t == 0.0:
        right = T[:, i0:i0 + width].copy()
    else:
        a = T[:, i0:i0 + width].astype(np.float64)
        b = T[:, i0 + 1:i0 + 1 + width].astype(np.float64)
        right = quantize((1.0 - t) * a + t * b)
    gt = np.full((height, width), s, np.float32)
    return left, right, gt


def _dot_pattern(rng, height, width, density=0.25, amplitude=180.0):
    dots = (rng.random((height + 2, width + 2)) < density).astype(np.float64)
    k = np.array([0.25, 0.5, 0.25])
    # separable ~1 px blob blur
    b = k[0] * dots[:, :-2] + k[1] * dots[:, 1:-1] + k[2] * dots[:, 2:]
    b = k[0] * b[:-2] + k[1] * b[1:-1] + k[2] * b[2:]
    return amplitude * b


def speckle_depth(width: int, height: int, rng: np.random.Generator):
    """Ground-truth depth (m) in the left view, plus the 'transparent' mask."""
    yy, xx = np.mgrid[0:height, 0:width].astype(np.float64)
    Z = np.full((height, width), 1.8)
    # slanted plane over a band of the image: depth 1.4 -> 0.7 left to right
    x0, x1 = 0.05 * width, 0.60 * width
    y0, y1 = 0.55 * height, 0.95 * height
    band = (xx >= x0) & (xx < x1) & (yy >= y0) & (yy < y1)
    Z[band] = 1.4 - 0.7 * (xx[band] - x0) / (x1 - x0)
    # 3-6 boxes (fronto-parallel rectangles) at 0.6-1.2 m
    for _ in range(int(rng.integers(3, 7))):
        w = rng.uniform(0.06, 0.18) * width
        h = rng.uniform(0.08, 0.25) * height
        bx = rng.uniform(0.0, width - w)
        by = rng.uniform(0.0, height - h)
        z = rng.uniform(0.6, 1.2)
        m = (xx >= bx) & (xx < bx + w) & (yy >= by) & (yy < by + h)
        Z[m] = np.minimum(Z[m], z)
    # one transparent disk (no projector pattern reaches the sensor)
    r = rng.uniform(0.06, 0.10) * min(width, height)
    cx = rng.uniform(r, width - r)
    cy = rng.uniform(r, height - r)
    disk = (xx - cx) ** 2 + (yy - cy) ** 2 < r * r
    Z[disk] = np.minimum(Z[disk], 1.0)
    return Z, disk


def speckle_pair(cfg: StereoConfig, frame_idx: int = 0, noise: bool = True):
    """D415-shaped active-stereo IR pair (see module docstring)."""
    rng = rng_for(frame_idx, cfg.tag)
    W, H = cfg.width, cfg.height
    Z, disk = speckle_depth(W, H, rng)
    disp = cfg.focal_px * cfg.baseline_m / Z                      # ground truth, left view
    ambient = 20.0
    left_clean = ambient + _dot_pattern(rng, H, W) * (~disk)
    # forward warp: left pixel x lands at xr = x - disp(x); per-segment linear map,
    # nearest surface (largest disparity) wins the z-buffer.
    u = np.arange(W)[None, :] - disp                               # [H][W]
    u0, u1 = u[:, :-1], u[:, 1:]
    d0, d1 = disp[:, :-1], disp[:, 1:]
    cont = np.abs(d1 - d0) <= 1.0                                  # same surface
    ys, xs, xr_all, dd, ss = [], [], [], [], []
    for j in (0, 1):
        xr = np.ceil(u0) + j
        ok = cont & (xr < u1) & (xr >= 0) & (xr < W) & (u1 > u0)
        t = np.where(ok, (xr - u0) / np.where(u1 > u0, u1 - u0, 1.0), 0.0)
        yi, xi = np.nonzero(ok)
        ys.append(yi); xs.append(xi); xr_all.append(xr[ok].astype(np.int64))
        dd.append((d0 + (d1 - d0) * t)[ok]); ss.append(xi + t[ok])
    ys = np.concatenate(ys); xr_all = np.concatenate(xr_all)
    dd = np.concatenate(dd); ss = np.concatenate(ss)
    order = np.lexsort((-dd, xr_all, ys))
    key = ys[order] * W + xr_all[order]
    first = np.ones(len(key), bool)
    first[1:] = key[1:] != key[:-1]
    sel = order[first]
    right_clean = np.full((H, W), ambient)                         # projector shadow
    sx = ss[sel]
    i0 = np.clip(np.floor(sx).astype(np.int64), 0, W - 2)
    t = sx - i0
    yr = ys[sel]
    right_clean[yr, xr_all[sel]] = (1 - t) * left_clean[yr, i0] + t * left_clean[yr, i0 + 1]
    if noise:
        left_n = apply_noise(left_clean, rng)
        right_n = apply_noise(right_clean, rng)
    else:
        left_n, right_n = left_clean, right_clean
    gt = disp.astype(np.float32)
    gt[disk] = np.nan
    return quantize(left_n), quantize(right_n), gt


def make_pair(cfg, frame_idx: int = 0):
    """(left u8[H][W], right u8[H][W], gt_disp f32[H][W]) for config A-E (or a StereoConfig)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if cfg.kind == "shift":
        return shift_pair(cfg.width, cfg.height, 7, frame_idx, cfg.tag)
    return speckle_pair(cfg, frame_idx)


def frame_pool(cfg, n: int):
    """n distinct frames of cfg stacked: (left u8[n][H][W], right u8[n][H][W])."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    L = np.empty((n, cfg.height, cfg.width), np.uint8)
    R = np.empty_like(L)
    for i in range(n):
        L[i], R[i], _ = make_pair(cfg, i)
    return L, R


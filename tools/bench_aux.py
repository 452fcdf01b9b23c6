"""Measurement of the auxiliary entry points at
config-C sizes on one B200: the sensor-noise front end, homography
rectification and depth registration.  CUDA events around K calls after W
warm-up calls; roofline = algorithmic bytes / time vs MEASURED_PEAKS.json's
HBM copy bandwidth (all three are streaming kernels).

    python tools/bench_aux.py [--frames 64] [--steps 10] [--warmup 3]

Prints one JSON line per entry point.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_11924_b200 as asd  # noqa: E402
import synth  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback B200_PROFILING.md"


def timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def line(name, frames, ms, alg_bytes, peak, src, extra):
    gbs = alg_bytes / (ms / 1e3) / 1e9
    return {"entry": name, "metric": "frames/s", "value": round(frames / (ms / 1e3), 1),
            "ms_per_call": round(ms, 4), "frames_per_call": frames,
            "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(gbs / peak, 4), "alg_bytes_per_call": alg_bytes, "peak_source": src},
            **extra}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    cfg = synth.CONFIGS["C"]
    H, W, n = cfg.height, cfg.width, args.frames
    peak, src = hbm_peak()
    dev = "cuda"
    rng = np.random.default_rng(0)

    # sensor noise: f32 clean in (4 B/px), u8 out (1 B/px)
    clean = torch.from_numpy(rng.uniform(0, 255, (n, H, W)).astype(np.float32)).to(dev)
    noisy = torch.empty(n, H, W, dtype=torch.uint8, device=dev)
    ms = timed(lambda: asd.sensor_noise(clean, 7, out=noisy), args.steps, args.warmup)
    print(json.dumps(line("asd_sensor_noise", n, ms, n * H * W * 5, peak, src,
                          {"config": "C images 1280x720, D415 noise (k=3.98, theta=0.254, mu=-0.231, "
                                     "sigma=0.83), fp64 Philox/Marsaglia-Tsang/Box-Muller"})))

    # rectification: u8 in (1 B/px, gathered), u8 out
    a = 0.01
    Hm = np.array([[np.cos(a), -np.sin(a), 2.5], [np.sin(a), np.cos(a), -1.5], [1e-6, 2e-6, 1.0]])
    rect = torch.empty_like(noisy)
    ms = timed(lambda: asd.rectify(Hm, noisy, out=rect), args.steps, args.warmup)
    print(json.dumps(line("asd_rectify", n, ms, n * H * W * 2, peak, src,
                          {"config": "C images 1280x720, rotation 0.01 rad + shift + mild perspective"})))

    # registration: f32 depth in (4 B/px), f32 out at 1920x1080 (fill 4 B, atomicMin 4 B per hit, finish 8 B)
    z = torch.from_numpy(rng.uniform(0.4, 2.0, (n, H, W)).astype(np.float32)).to(dev)
    ir = (W, H, float(cfg.focal_px), float(cfg.focal_px), (W - 1) / 2, (H - 1) / 2)
    rgb = (1920, 1080, 1380.0, 1380.0, 959.5, 539.5)
    out = torch.empty(n, 1080, 1920, device=dev)
    eye = np.eye(3, dtype=np.float32)
    ms = timed(lambda: asd.register_depth(ir, rgb, eye, [-0.015, 0.0, 0.0], z, out=out), args.steps, args.warmup)
    alg = n * (H * W * (4 + 4) + 1920 * 1080 * (4 + 8))
    print(json.dumps(line("asd_register_depth", n, ms, alg, peak, src,
                          {"config": "C depth 1280x720 -> RGB 1920x1080 (Table II output size), "
                                     "15 mm baseline offset"})))


if __name__ == "__main__":
    main()

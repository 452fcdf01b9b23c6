#!/usr/bin/env python3
"""Small cases of every kernel family, each checked against the oracle by
per-frame checksum and valid count, for the checked build (tools/checked.sh:
-DASD_CHECKED = index asserts that trap, poisoned scratch, pseudo-random
__nanosleep jitter at every synchronisation point; compute-sanitizer is closed
on the GPU pool) and, where available, compute-sanitizer.

    ASD_LIB=paper_2201_11924_b200/lib/variants/checked.so python tools/sanitize_cases.py --repeat 20

The cases cover the D3 cluster sweeps (DSMEM halos, relaxed cluster arrive,
cp.async census ring in K_down, TMA/mbarrier ring in K_up) at cluster sizes > 1
for the D = 64 (T = 2) and D = 128 (T = 4, the config-C instance) layouts, the
row and WTA kernels, the SGBM and R2 variants, the multi-slot D3 pipeline
(max_batch > group) and engine D1.  Exit code 1 on any oracle mismatch.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2201_11924_b200 as asd  # noqa: E402
import synth  # noqa: E402


def _cfg(name, **over):
    d = synth.CONFIGS[name].params_dict()
    d.update(over)
    return d


def _pairs(d, n, tag):
    """n seeded speckle pairs at the size of d (synthetic scene recipe)."""
    cfg = synth.StereoConfig("S", d["width"], d["height"], d["num_disp"], d["census_w"], d["census_h"],
                             d["paths"], d["focal_px"], tag=tag)
    Ls, Rs = [], []
    for i in range(n):
        L, R, _ = synth.speckle_pair(cfg, i)
        Ls.append(L)
        Rs.append(R)
    return np.stack(Ls), np.stack(Rs)


# name -> (params, frames, max_batch, group or None)
def cases():
    small128 = dict(width=256, height=64, num_disp=128, min_disp=0, census_w=9, census_h=7, paths=8,
                    focal_px=260.0)
    small64 = dict(width=160, height=120, num_disp=64, min_disp=0, census_w=7, census_h=7, paths=8,
                   focal_px=160.0)
    return {
        "A_d3": (_cfg("A", engine=3), 3, 2, 1),
        "A_d1": (_cfg("A", engine=1), 2, 2, None),
        "s64_d3": ({**_cfg("C"), **small64, "engine": 3}, 3, 2, 1),
        "s128_d3": ({**_cfg("C"), **small128, "engine": 3}, 3, 2, 1),
        "s128_d3_sgbm": ({**_cfg("C"), **small128, "engine": 3, "block_w": 3, "block_h": 3,
                          "p1": 72, "p2": 288}, 2, 2, 1),
        "s128_d3_r2": ({**_cfg("C"), **small128, "engine": 3, "lr_mode": 1}, 2, 2, 1),
        "s128_d3_med": ({**_cfg("C"), **small128, "engine": 3, "median_ksize": 5}, 2, 2, 1),
        "s64_d1": ({**_cfg("C"), **small64, "engine": 1}, 2, 2, None),
        "B_d3": (_cfg("B", engine=3), 2, 2, 1),
        # config C in bench.py's pipeline: 24 frames over two 11-frame slots
        # (groups 11, 11, 2), 4 distinct frames
        "C_d3": (_cfg("C", engine=3), 24, 22, None),
        # frames wider than one cluster: two clusters joined through global
        # memory (segment-boundary counters), D = 128 and D = 256
        "seg128_d3": ({**_cfg("C"), "width": 2100, "height": 40, "focal_px": 430.0 * 2100 / 424,
                       "engine": 3}, 4, 4, None),
        "seg256_d3": ({**_cfg("C"), "width": 1100, "height": 48, "num_disp": 256,
                       "focal_px": 430.0 * 1100 / 424 * 2, "engine": 3}, 4, 4, None),
        # two clusters, census staged by cp.async (width not a multiple of 4)
        "seg128_cpa_d3": ({**_cfg("C"), "width": 2102, "height": 32, "focal_px": 430.0 * 2102 / 424,
                           "engine": 3}, 3, 3, None),
        # four clusters per frame (middle segments receive from both sides)
        "seg4_256_d3": ({**_cfg("C"), "width": 2300, "height": 32, "num_disp": 256,
                         "focal_px": 430.0 * 2300 / 424 * 2, "engine": 3}, 3, 3, None),
    }


def run(name, d, n, mb, group, repeat=1):
    import torch
    pool = min(n, 4)
    L0, R0 = _pairs(d, pool, tag=97)
    L, R = L0[[i % pool for i in range(n)]], R0[[i % pool for i in range(n)]]
    H, W = d["height"], d["width"]
    Lg, Rg = torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()
    disp = torch.empty(n, H, W, device="cuda")
    depth = torch.empty_like(disp)
    stats = torch.zeros(n, 4, dtype=torch.int32, device="cuda")
    t0 = time.time()
    with asd.Stereo(asd.Params(**d), 0, mb) as st:
        if group and st.engine == 3:
            st.group = group
        runs = []
        for _ in range(repeat):
            stats.zero_()
            st.asd_depth_batch(Lg, Rg, disp, depth, stats)
            torch.cuda.synchronize()
            runs.append(stats.cpu().numpy().copy())
        info = st.plan_info
    gpu_s = time.time() - t0
    p = oracle.Params(**{k: v for k, v in d.items() if k != "engine"})
    res = {}

    def orc(i):
        o = oracle.compute(p, L0[i], R0[i])
        res[i] = (oracle.checksum(o["dstar_l"], o["mask"]), int((o["mask"] == 0).sum()))

    import threading
    ths = [threading.Thread(target=orc, args=(i,)) for i in range(pool)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    bad = 0
    for s in runs:
        for i in range(n):
            h, v = res[i % pool]
            if (int(s[i, 0]) & 0xFFFFFFFF) != h or int(s[i, 1]) != v:
                bad += 1
    print(f"{name}: frames={n} x {repeat} runs max_batch={mb} group={group} gpu_s={gpu_s:.1f} "
          f"mismatches={bad} [{info}]", flush=True)
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--repeat", type=int, default=1, help="runs of each batch (checked builds: jitter)")
    a = ap.parse_args()
    bad = 0
    print(f"library: {asd.abi.LIB_PATH}", flush=True)
    for name, (d, n, mb, g) in cases().items():
        if a.only and name not in a.only.split(","):
            continue
        bad += run(name, d, n, mb, g, a.repeat)
    print("SANITIZE_CASES", "FAIL" if bad else "OK", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()

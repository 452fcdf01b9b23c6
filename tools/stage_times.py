"""Per-stage device times (libasd live CUDA-event timing) for one configuration.

    python tools/stage_times.py [--config C] [--paths 8] [--frames 32] [--max-batch 32] [--engine 0]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2201_11924_b200 as asd
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C")
ap.add_argument("--paths", type=int, default=None)
ap.add_argument("--frames", type=int, default=32)
ap.add_argument("--max-batch", type=int, default=0)
ap.add_argument("--engine", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--timeline", action="store_true", help="print the per-launch timeline")
ap.add_argument("--group", type=int, default=0, help="D3 pipeline group (frames); 0 = default")
ap.add_argument("--block", type=int, default=1, help="SGBM block (P1/P2 scaled by its area)")
ap.add_argument("--lr-mode", type=int, default=0)
ap.add_argument("--width", type=int, default=0, help="override the configuration's width (synthetic scene rescaled)")
ap.add_argument("--height", type=int, default=0)
args = ap.parse_args()
cfg = synth.CONFIGS[args.config]
if args.width or args.height:
    w, h = args.width or cfg.width, args.height or cfg.height
    cfg = synth.StereoConfig(cfg.name + "'", w, h, cfg.num_disp, cfg.census_w, cfg.census_h, cfg.paths,
                             cfg.focal_px * w / cfg.width, tag=cfg.tag)
d = cfg.params_dict()
if args.paths:
    d["paths"] = args.paths
if args.block > 1:
    a2 = args.block * args.block
    d.update(block_w=args.block, block_h=args.block, p1=8 * a2, p2=32 * a2)
if args.lr_mode:
    d["lr_mode"] = args.lr_mode
Lp, Rp = synth.frame_pool(cfg, 4)
idx = [i % 4 for i in range(args.frames)]
L = torch.from_numpy(Lp[idx]).cuda(); R = torch.from_numpy(Rp[idx]).cuda()
out = torch.empty(args.frames, cfg.height, cfg.width, device="cuda")
if args.max_batch <= 0:
    probe = asd.Stereo(asd.Params(**d, engine=args.engine), 0, 1)
    fpw = probe.frames_per_wave
    probe.close()
    args.max_batch = max(1, (32 // fpw) * fpw) if fpw > 0 else 32
    print("frames per wave", fpw, "max_batch", args.max_batch)
st = asd.Stereo(asd.Params(**d, engine=args.engine), 0, args.max_batch)
if args.group > 0 and st.engine == 3:
    st.group = args.group
print(st.plan_info, "group", st.group)
st.asd_depth_batch(L, R, out, out)
torch.cuda.synchronize()
st.profile_begin(4096)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.reps):
    st.asd_depth_batch(L, R, out, out)
e1.record()
torch.cuda.synchronize()
wall = e0.elapsed_time(e1)
tl = st.profile_timeline(4096) if args.timeline else []
prof = st.profile_end()
n = args.frames * args.reps
tot = sum(prof[k]["ms"] for k in asd.abi.STAGES)
print(f"config {args.config} paths {d['paths']} engine {st.engine}: {1000 * tot / n:.1f} us/frame "
      f"sum of stages, {1000 * wall / n:.1f} us/frame wall, {n / (wall / 1000):.0f} frames/s")
for name, a, b in tl:
    print(f"  {name:7s} {a:9.3f} {b:9.3f}  {b - a:7.3f} ms")
for k in asd.abi.STAGES:
    if prof[k]["launches"]:
        us = 1000 * prof[k]["ms"] / n
        gbs = prof[k]["alg_bytes"] / (prof[k]["ms"] / 1000) / 1e9
        print(f"  {k:7s} {us:8.1f} us/frame  {gbs:8.1f} GB/s algorithmic  launches {prof[k]['launches']}")

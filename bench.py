#!/usr/bin/env python3
"""Benchmark of the active-stereo depth path (arXiv 2201.11924 "SimSense" stage).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl asd|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)

A step = one pass of the whole hot path (census -> Hamming cost -> 8-path SGM ->
WTA/uniqueness -> sub-pixel -> right view -> LR -> depth) over a batch of
FRAMES_PER_STEP synthetic config-C frames (1280x720, D=128, census 9x7, 8-path;
BASELINE.json configs[2], the configuration its metric is quoted on) per GPU.
Frames are independent, so ranks shard frames with no data-path collective
(weak scaling); NCCL only all-reduces the timer and all-gathers per-frame stats
after the timed region.  Rank 0 prints ONE JSON line.

--impl reference times the CPU oracle (oracle/, plain C) on the host cores, one
full config-C frame per worker thread per step: the only reference this
paper-only tier has (no upstream code exists).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/s and Gcell/s (W·H·D) at 1280×720×D128 8-path; HBM GB/s vs peak"
CONFIG = "C"
METRIC_D = "frames/s and Gcell/s (W·H·D) at 1920×1080×D256 8-path (config D); HBM GB/s vs peak"
FRAMES_PER_STEP = 128          # inputs 128 x 2 x 0.92 MB = 236 MB per step > 126 MB L2
POOL = 8                       # distinct synthetic frames (kernels are data-oblivious)
CRITICAL = ("census", "block", "down", "up")   # D3 stages on the high-priority streams (s_cen, s_hi)
MAX_BATCH = 33                 # frames in flight: three D3 waves (three scratch slots: e2e 1836 -> 1900 vs two)


KERNEL_NAMES = {"census": "census_kernel (K1)", "dir": "sgm_dir_kernel (D1, one path direction)",
                "wta": "WTA kernel (K4: D1 wta_kernel / D3 wta2_kernel)", "lr": "lr_depth_kernel (K5)",
                "down": "vsweep_kernel<down> (D3, 3 downward paths)",
                "up": "vsweep_kernel<up> (D3, 3 upward paths)",
                "row": "hrow_kernel (D3, horizontal paths)",
                "block": "block_cost_kernel (SGBM block cost volume)"}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


# ----------------------------------------------------------------- clocks
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


class ClockSampler:
    """nvidia-smi sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                s, m, r = float(parts[0]), float(parts[1]), int(parts[2], 16)
            except ValueError:
                continue
            sm.append(s)
            mx = max(mx, m)
            for bit, name in REASONS.items():
                if r & bit and name != "gpu_idle":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def run_params(cfg, block: int, lr_mode: int = 0, median: int = 0, engine: int = 0) -> dict:
    """Config parameters; block > 1 = SGBM with P1 = 8*area, P2 = 32*area;
    lr_mode 1 = the R2 right view (reading c24); median = median ksize (c20);
    engine 0 = auto, 1 = D1, 3 = D3."""
    d = cfg.params_dict()
    if engine:
        d.update(engine=engine)
    if block > 1:
        d.update(block_w=block, block_h=block, p1=8 * block * block, p2=32 * block * block)
    if lr_mode:
        d.update(lr_mode=lr_mode)
    if median:
        d.update(median_ksize=median)
    return d


def bench_config(args, world: int) -> dict:
    """The `config` object, identical in both arms (GPU and reference) of the
    same command line: the workload and the L2 statement (run details go under
    `run`)."""
    import synth
    cfg = synth.CONFIGS[args.config]
    B = args.job // max(1, world) if args.job else args.frames
    return {"workload": workload(args.block, args.lr_mode, args.median, args.config)
                        + (f" (P2={args.p2})" if args.p2 else "")
                        + (f"; E: job of {args.job} frames per step sharded over {world} GPU(s)" if args.job else ""),
            "l2": f"inputs larger than L2 ({2 * B * cfg.height * cfg.width / 1e6:.0f} MB/step/GPU) "
                  "+ per-frame scratch > L2"}


def host_context(params, cpu) -> dict:
    """SURVEY §8(d)'s oracle context in the same run: the host CPU, the oracle's
    single-frame latency per config (A and B timed here on one core; C from the
    cpu_baseline run, one frame per thread), and the paper's Table II numbers
    with their hardware (another workload and GPU: context only)."""
    import oracle
    import synth
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    lat = {}
    for name in ("A", "B"):
        c = synth.CONFIGS[name]
        L, R, _ = synth.make_pair(name, 0)
        t0 = time.perf_counter()
        oracle.compute(oracle.Params(**c.params_dict()), L, R)
        lat[name] = round(time.perf_counter() - t0, 3)
    if cpu:
        lat["C"] = cpu.get("frame_latency_s")
    return {"cpu_model": model, "host_cores": len(os.sched_getaffinity(0)),
            "oracle_single_frame_latency_s": lat,
            "paper_table2": {"hardware": "1x RTX 4090 (P:296); OpenCV SGBM on i5-10400",
                             "workload": "960x540 -> 1920x1080, 4-path, median 3 (not config C)",
                             "sgm_fps": {str(k): v[0] for k, v in TABLE2_FPS.items()},
                             "sgbm_fps": {str(k): v[1] for k, v in TABLE2_FPS.items()},
                             "source": "PAPER.md Table II, BASELINE.md §1"}}


def workload(block: int, lr_mode: int = 0, median: int = 0, cfg_name: str = "C") -> str:
    extra = (", R2 right view" if lr_mode else "") + (f", median {median}" if median else "")
    if cfg_name == "D":
        return ("D: 1920x1080, D=256, census 9x7, P1=8 P2=32, 8-path SGM, uniqueness 10%, LR 1 px, "
                "sub-pixel, depth (cost-volume-pressure stress)" + extra)
    if block > 1:
        a = block * block
        return (f"C-SGBM{block}x{block}: 1280x720, D=128, census 9x7, {block}x{block} block, "
                f"P1={8 * a} P2={32 * a}, 8-path SGM, uniqueness 10%, LR 1 px, sub-pixel, depth" + extra)
    return ("C: 1280x720, D=128, census 9x7, P1=8 P2=32, 8-path SGM, uniqueness 10%, LR 1 px, "
            "sub-pixel, depth" + extra)


# ----------------------------------------------------------------- oracle (CPU)
def oracle_workers(params: dict | None = None):
    """Host threads for the oracle: all cores, at most 32, and as many frames as
    fit in half the free host memory (the oracle holds ~13 B per cell: the u8
    cost, u32 block cost and u32 aggregate volumes)."""
    cores = len(os.sched_getaffinity(0))
    cells = 1280 * 720 * 128
    if params:
        cells = params["width"] * params["height"] * params["num_disp"]
    try:
        import psutil
        mem_frames = int(0.5 * psutil.virtual_memory().available // (13.0 * cells + 64e6))
    except Exception:
        mem_frames = 8
    return max(1, min(cores, mem_frames, 32)), cores


def oracle_params(params: dict):
    """oracle.Params of a run's parameters (the engine choice is the GPU's alone)."""
    import oracle
    return oracle.Params(**{k: v for k, v in params.items() if k != "engine"})


def oracle_frames_parallel(params, Ls, Rs, nworkers):
    """The oracle as it stands: one full frame per worker thread (ctypes releases
    the GIL, so the C oracle runs on nworkers host cores)."""
    import oracle
    p = oracle_params(params)
    oracle.lib()
    out = [None] * nworkers

    def run(i):
        out[i] = oracle.compute(p, Ls[i % len(Ls)], Rs[i % len(Rs)])

    ths = [threading.Thread(target=run, args=(i,)) for i in range(nworkers)]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return time.perf_counter() - t0, out


def _oracle_sig(o) -> tuple:
    """(checksum, valid count) of one oracle frame -- the per-frame statistics
    the library's asd_frame_stats carries (SURVEY §8(e) checksum)."""
    import oracle
    return (oracle.checksum(o["dstar_l"], o["mask"]), int((o["mask"] == 0).sum()))


def cpu_baseline(params, Ls, Rs, cfg_name="C"):
    """The oracle timed on the host cores (one full frame per thread); also
    returns the (checksum, valid) of every pool frame it computed, which the
    parity check of the GPU frames reuses."""
    nworkers, cores = oracle_workers(params)
    wall, outs = oracle_frames_parallel(params, Ls, Rs, nworkers)
    sigs = {i % len(Ls): _oracle_sig(o) for i, o in enumerate(outs)}
    return {"value": round(nworkers / wall, 4), "unit": "frames/s", "cores": nworkers,
            "kind": "oracle", "frame_latency_s": round(wall, 2),
            "sample": f"{nworkers} full config-{cfg_name} frames"
                      f"{' (SGBM block)' if params.get('block_w', 1) > 1 else ''}, one per host thread "
                      f"on {nworkers} of {cores} cores, plain-C oracle (gcc -O2), wall {wall:.1f} s"}, sigs


def oracle_pool_sigs(params, Ls, Rs, have: dict | None = None) -> dict:
    """(checksum, valid) of every frame of the pool, by the oracle (frames not in
    `have` are computed, one per host thread, memory-bounded)."""
    import oracle
    sigs = dict(have or {})
    todo = [i for i in range(len(Ls)) if i not in sigs]
    if not todo:
        return sigs
    nworkers, _ = oracle_workers(params)
    p = oracle_params(params)
    oracle.lib()
    for k in range(0, len(todo), nworkers):
        part = todo[k:k + nworkers]
        res = {}

        def run(i):
            res[i] = _oracle_sig(oracle.compute(p, Ls[i], Rs[i]))

        ths = [threading.Thread(target=run, args=(i,)) for i in part]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        sigs.update(res)
    return sigs


def parity_check(stats, frame_ids, sigs) -> dict:
    """Every GPU frame's (checksum, valid) against the oracle's for the same
    input (frame f is pool[f % POOL]).  stats: int array [n, 4]."""
    bad = []
    for row, f in zip(stats, frame_ids):
        cs, valid = sigs[f % POOL]
        if (int(row[0]) & 0xFFFFFFFF) != cs or int(row[1]) != valid:
            bad.append(int(f))
    return {"frames": len(frame_ids), "mismatches": len(bad), "first_bad": bad[:8],
            "oracle_frames": len(sigs), "check": "per-frame (checksum of d* and mask, valid count) == oracle"}


def run_reference(args):
    """--impl reference: the CPU oracle timed as the reference arm (rank 0 only)."""
    import synth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    params = run_params(cfg, args.block, args.lr_mode, args.median)
    if args.p2:
        params["p2"] = args.p2
    Ls, Rs = synth.frame_pool(cfg, min(POOL, 4))
    nworkers, cores = oracle_workers(params)
    for _ in range(args.warmup):
        oracle_frames_parallel(params, Ls, Rs, nworkers)
    tot = 0.0
    for _ in range(args.steps):
        w, _ = oracle_frames_parallel(params, Ls, Rs, nworkers)
        tot += w
    frames = nworkers * args.steps
    value = frames / tot
    line = {"impl": "reference", "metric": METRIC if args.config == "C" else METRIC_D, "value": round(value, 4), "unit": "frames/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000 * tot / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u16", "data": "synthetic",
            "gcells_per_s": round(value * cfg.cells / 1e9, 6),
            "config": bench_config(args, int(os.environ.get("WORLD_SIZE", str(args.gpus)))),
            "run": {"frames_per_step": nworkers, "impl": "CPU oracle (oracle/asd_oracle.c)",
                    "note": "each step: one full frame of the workload per host thread (a bounded sample)"},
            "cpu_baseline": {"value": round(value, 4), "unit": "frames/s", "cores": nworkers,
                             "kind": "oracle",
                             "sample": f"{nworkers} full config-C frames per step, one per thread "
                                       f"({nworkers} of {cores} cores)"},
            "e2e": {"value": round(value, 4), "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------ the paper's Table II workload
TABLE2_FPS = {64: (414.51, 342.24), 96: (326.79, 268.98), 128: (281.26, 232.49), 256: (147.13, 128.56)}


def d1_gate(asd, params, L, R, dev, hbm_peak, steps: int = 2, frames: int = 32, traffic_ok: bool = True):
    """North-star gate: the aggregation kernel of engine D1 (sgm_dir_kernel, one
    path direction per launch, u16 S read-modify-write = 4 B/cell, HBM-bound by
    design) against the HBM roofline, measured live on the same frames: its
    average launch duration from the library's CUDA events on the launching
    stream, algorithmic bytes / duration.  D1 runs the whole
    path (census, 8 directions, WTA, LR/depth) serially; fps is that engine's."""
    import torch
    n = min(frames, L.shape[0])
    d = dict(params, engine=1)
    st = asd.Stereo(asd.Params(**d), dev.index, n)
    Lg, Rg = L[:n].contiguous(), R[:n].contiguous()
    disp = torch.empty(n, L.shape[1], L.shape[2], device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(2):
        st.asd_depth_batch(Lg, Rg, disp, disp, None, stream=stream)
    torch.cuda.synchronize(dev)
    st.profile_begin(4096)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        st.asd_depth_batch(Lg, Rg, disp, disp, None, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    prof = st.profile_end()
    st.close()
    ms = e0.elapsed_time(e1)
    dp = prof["dir"]
    avg = dp["ms"] / max(1, dp["launches"])
    alg = dp["alg_bytes"] / max(1, dp["launches"])
    ach = alg / (avg / 1e3) / 1e9
    traffic = None          # ncu dram bytes per launch (profiles/ncu_traffic.json "dir": per frame, all 8 directions averaged)
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if traffic_ok and os.path.exists(tpath):
        try:
            per_frame = json.load(open(tpath)).get("dir")
            traffic = per_frame * n if per_frame is not None else None
        except Exception:
            traffic = None
    return {"kernel": "sgm_dir_kernel (engine D1, one path direction per launch)", "bound": "hbm", "traffic": traffic,
            "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s", "frac": round(ach / hbm_peak, 4),
            "target_frac": 0.6, "alg_bytes_per_launch": alg, "avg_launch_ms": round(avg, 4),
            "launches": dp["launches"], "engine_fps": round(n * steps / (ms / 1e3), 1),
            "note": "all 8 directions averaged; 2 B/cell for the first (write-only), 4 B/cell for the others"}


def run_table2(args):
    """--table2 D: the paper's own benchmark (Table II):
    960x540 IR pair -> 4-path SGM (or SGBM with --block) with uniqueness,
    sub-pixel, LR, median 3 and depth, registered to a 1920x1080 RGB frame
    (reading c16).  One step = a batch of frames through asd_depth_batch +
    asd_register_depth; e2e adds the H2D of the pair and the D2H of the
    registered depth.  vs_baseline = value / the paper's RTX 4090 FPS for the
    same D (another GPU: context for the like-for-like workload)."""
    import numpy as np
    import torch
    import paper_2201_11924_b200 as asd
    import synth
    D = args.table2
    cfg = synth.CONFIGS[f"T{D}"]
    params = run_params(cfg, args.block, args.lr_mode, 3, args.engine)
    B, H, W = args.frames, cfg.height, cfg.width
    dev = torch.device("cuda", 0)
    pool_L, pool_R = synth.frame_pool(cfg, POOL)
    idx = [f % POOL for f in range(B)]
    Lh = torch.from_numpy(pool_L[idx]).pin_memory()
    Rh = torch.from_numpy(pool_R[idx]).pin_memory()
    L, R = Lh.to(dev), Rh.to(dev)
    disp = torch.empty(B, H, W, device=dev)
    depth = torch.empty_like(disp)
    reg = torch.empty(B, 1080, 1920, device=dev)
    regh = torch.empty(B, 1080, 1920).pin_memory()
    ir = (W, H, float(cfg.focal_px), float(cfg.focal_px), (W - 1) / 2, (H - 1) / 2)
    rgb = (1920, 1080, 2.0 * float(cfg.focal_px), 2.0 * float(cfg.focal_px), 959.5, 539.5)
    eye, t = np.eye(3, dtype=np.float32), [-0.015, 0.0, 0.0]          # D415-like RGB offset
    probe = asd.Stereo(asd.Params(**params), 0, 1)
    fpw = probe.frames_per_wave
    probe.close()
    mb = max(1, (MAX_BATCH // fpw) * fpw) if fpw > 0 else MAX_BATCH
    st = asd.Stereo(asd.Params(**params), 0, mb)
    stream = torch.cuda.current_stream(dev)

    def step():
        st.asd_depth_batch(L, R, disp, depth, None, stream=stream)
        asd.register_depth(ir, rgb, eye, t, depth, out=reg, stream=stream)

    def step_e2e():
        L.copy_(Lh, non_blocking=True)
        R.copy_(Rh, non_blocking=True)
        step()
        regh.copy_(reg, non_blocking=True)

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1)

    with ClockSampler(0) as clk:
        ms = timed(step)
    ms_e2e = timed(step_e2e)
    value = B * args.steps / (ms / 1e3)
    paper = TABLE2_FPS[D][1 if args.block > 1 else 0]
    line = {"metric": f"SimSense {'SGBM' if args.block > 1 else 'SGM'} FPS, Table II workload "
                      f"(960x540 -> 1920x1080, 4-path, D={D})",
            "value": round(value, 2), "unit": "frames/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": round(value / paper, 2), "dtype": "u16", "data": "synthetic",
            "config": {"workload": f"T{D}: 960x540, D={D}, census 9x7, P1={params['p1']} P2={params['p2']}, "
                                   f"4-path SGM{' block %dx%d' % (args.block, args.block) if args.block > 1 else ''}, "
                                   "uniqueness 10%, LR 1 px, sub-pixel, median 3, depth, registration to 1920x1080",
                       "frames_per_step": B, "engine": st.plan_info,
                       "paper": {"fps": paper, "hardware": "1x RTX 4090 (P:296)", "source": "PAPER.md Table II"}},
            "clocks": clk.summary(),
            "e2e": {"value": round(B * args.steps / (ms_e2e / 1e3), 2), "unit": "frames/s",
                    "h2d_bytes_per_step": int(Lh.numel() + Rh.numel()), "d2h_bytes_per_step": int(4 * regh.numel()),
                    "api": "asd_depth_batch + asd_register_depth, torch pinned copies"}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm
# Integer lane-ops per cell of each D3 kernel: SURVEY §8(d)'s model (o = 5.5
# packed u16x2 lane-ops per cell-path of the recursion, + 2 per cell where the
# Hamming cost is evaluated; the library reports these as alg_ops) and the
# minimal packed model of DESIGN.md §5 (2.5 per cell-path, 3 per cell of cost).
def op_models(stage: str, paths: int, blk: bool):
    np_ = 3 if paths == 8 else 1
    c8, cmin = (0.0, 0.0) if blk else (2.0, 3.0)
    return {"down": (np_ * 5.5 + c8, np_ * 2.5 + cmin), "up": (np_ * 5.5, np_ * 2.5 + 2.0),
            "row": (2 * 5.5 + c8, 2 * 2.5 + cmin + 2.0)}.get(stage)


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch this command as N ranks
    (one per GPU, NCCL) under torch.distributed.run on 127.0.0.1."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA device(s) visible"}), flush=True)
        return 2
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def gather_and_check(stats, ms: float, sigs_fn, device=None):
    """After the timed region: max of the timer over ranks (all_reduce MAX) and
    all_gather of the per-frame stats (NCCL on GPUs, gloo in the CPU test); on
    rank 0 every gathered frame's (checksum, valid) is compared with the
    oracle's (sigs_fn() -> {pool index: (checksum, valid)}).  Shards are
    contiguous and equal, so the gathered row i is global frame i.  Returns
    (ms_max, all_stats [frames, 4] int numpy, parity dict or None off rank 0)."""
    import torch.distributed as dist
    from paper_2201_11924_b200.dist import gather_frame_stats, max_over_ranks
    ms_max = max_over_ranks(ms, device)
    allst = gather_frame_stats(stats).cpu().numpy()
    rank = dist.get_rank() if dist.is_available() and dist.is_initialized() else 0
    if rank != 0:
        return ms_max, allst, None
    return ms_max, allst, parity_check(allst, list(range(len(allst))), sigs_fn())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="asd", choices=["asd", "reference"])
    ap.add_argument("--frames", type=int, default=FRAMES_PER_STEP, help="frames per step per GPU")
    ap.add_argument("--max-batch", type=int, default=0,
                    help="frames in flight (0: a whole number of cluster waves, ~33 = 3 slots at config C)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-gate", action="store_true", help="skip the D1 aggregation-kernel HBM gate measurement")
    ap.add_argument("--no-parity", action="store_true", help="skip the per-frame oracle check (profiling runs)")
    ap.add_argument("--job", type=int, default=0,
                    help="config E: a fixed job of this many frames per step (e.g. 4096), frame-sharded over the ranks (strong scaling)")
    ap.add_argument("--block", type=int, default=1,
                    help="SGBM block size (odd; 1 = SGM, the headline line)")
    ap.add_argument("--lr-mode", type=int, default=0, help="right view: 0 = R1 (headline), 1 = R2")
    ap.add_argument("--median", type=int, default=0, help="median ksize 0 / 3 / 5")
    ap.add_argument("--table2", type=int, default=0, choices=[0, 64, 96, 128, 256],
                    help="the paper's Table II workload at this max disparity (not the headline line)")
    ap.add_argument("--engine", type=int, default=0, choices=[0, 1, 3],
                    help="0 = auto (D3 where its envelope allows), 1 = D1 (per-direction, HBM-bound), 3 = D3")
    ap.add_argument("--config", default=CONFIG, choices=["C", "D"],
                    help="C = the headline 1280x720 D=128 line; D = 1920x1080 D=256")
    ap.add_argument("--p2", type=int, default=0, help="override P2 (e.g. 40: outside the 16-bit-key envelope)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.table2:
        return run_table2(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2201_11924_b200 as asd
    import synth
    from paper_2201_11924_b200.dist import shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    cfg = synth.CONFIGS[args.config]
    params = run_params(cfg, args.block, args.lr_mode, args.median, args.engine)
    if args.p2:
        params["p2"] = args.p2
    H, W = cfg.height, cfg.width
    pool_L, pool_R = synth.frame_pool(cfg, POOL)
    if args.job:
        # config E: one fixed job of args.job frames per step, frame-sharded across the
        # ranks; total work fixed as N grows -> strong scaling
        if args.job % world:
            raise SystemExit(f"--job {args.job} must divide evenly over {world} ranks (stats all_gather)")
        f0, f1 = shard_range(args.job, rank, world)
        B = f1 - f0
        args.no_e2e = True          # pinned host copies of a 4096-frame job exceed the host budget
    else:
        B = args.frames
        f0, f1 = shard_range(world * B, rank, world)      # this rank's frames of the job
    idx = [f % POOL for f in range(f0, f1)]
    L = torch.from_numpy(pool_L[idx]).to(dev)
    R = torch.from_numpy(pool_R[idx]).to(dev)
    disp = torch.empty(B, H, W, device=dev)
    depth = torch.empty(B, H, W, device=dev)
    stats = torch.zeros(B, 4, dtype=torch.int32, device=dev)
    if args.max_batch <= 0:
        probe = asd.Stereo(asd.Params(**params), local, 1)
        fpw = probe.frames_per_wave
        probe.close()
        args.max_batch = max(1, (MAX_BATCH // fpw) * fpw) if fpw > 0 else MAX_BATCH
    st = asd.Stereo(asd.Params(**params), local, args.max_batch)
    stream = torch.cuda.current_stream(dev)

    def step():
        st.asd_depth_batch(L, R, disp, depth, stats, stream=stream)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---- timed region: K steps, CUDA events on the launching stream, no
    # instrumentation inside (the per-stage profile is a separate pass below)
    lp = st.launches_per_batch(B)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats.zero_()
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
    ms = e0.elapsed_time(e1)
    stats_timed = stats.clone()                 # the last timed step's per-frame stats

    # ---- profiled pass (library CUDA events around every launch): stage_ms,
    # the dominant kernel's average launch time, the pipeline timeline
    psteps = max(1, min(args.steps, 3))
    st.profile_begin(max_launches=lp * psteps + 16)
    for _ in range(psteps):
        step()
    torch.cuda.synchronize(dev)
    timeline = st.profile_timeline(lp * psteps + 16)
    prof = st.profile_end()
    frames_total = (args.job if args.job else world * B) * args.steps

    # ---- end-to-end through the host entry point (pinned host buffers)
    e2e, sh = None, None
    if not args.no_e2e:
        Lh = torch.from_numpy(pool_L[idx]).pin_memory()
        Rh = torch.from_numpy(pool_R[idx]).pin_memory()
        dh = torch.empty(B, H, W).pin_memory()
        zh = torch.empty(B, H, W).pin_memory()
        sh = torch.zeros(B, 4, dtype=torch.int32).pin_memory()
        for _ in range(max(1, args.warmup)):
            st.asd_depth_batch_host(Lh, Rh, dh, zh, sh, stream=stream)
        barrier()
        torch.cuda.synchronize(dev)
        sh.zero_()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        for _ in range(args.steps):
            st.asd_depth_batch_host(Lh, Rh, dh, zh, sh, stream=stream)
        h1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        from paper_2201_11924_b200.dist import max_over_ranks
        t2 = max_over_ranks(h0.elapsed_time(h1), dev)
        e2e = {"value": round(frames_total / (t2 / 1000.0), 3), "unit": "frames/s",
               "h2d_bytes_per_step": int(Lh.numel() + Rh.numel()),
               "d2h_bytes_per_step": int(4 * (dh.numel() + zh.numel()) + 16 * B),
               "api": "asd_depth_batch_host"}

    # ---- stats gather (NCCL, after timing) + per-frame parity vs the oracle
    cpu = None
    sigs_cache = {}

    def sigs_fn():
        nonlocal cpu
        if not sigs_cache:
            have = {}
            if world == 1 and not args.no_cpu_baseline:
                cpu, have = cpu_baseline(params, pool_L, pool_R, args.config)
            sigs_cache.update(oracle_pool_sigs(params, pool_L, pool_R, have))
        return sigs_cache

    no_sigs = (lambda: {i: (0, 0) for i in range(POOL)})
    ms_max, st_all, parity = gather_and_check(stats_timed, ms, no_sigs if args.no_parity else sigs_fn, dev)
    parity_e2e = None
    if sh is not None:
        sh_dev = sh.to(dev)
        _, _, parity_e2e = gather_and_check(sh_dev, 0.0, no_sigs if args.no_parity else sigs_fn, dev)
    value = frames_total / (ms_max / 1000.0)

    if rank == 0:
        if world == 1 and not args.no_cpu_baseline and cpu is None:
            cpu, _ = cpu_baseline(params, pool_L, pool_R, args.config)
        pk = peaks()
        hbm_peak = pk["hbm_gbs"] if pk else 6650.0
        sm_mhz = pk.get("sm_max_mhz", 1965.0) if pk else 1965.0
        nsm = torch.cuda.get_device_properties(dev).multi_processor_count
        alu_peak = nsm * 128 * sm_mhz * 1e6 / 1e12       # T int lane-ops/s
        # Dominant kernel: D3 runs the census/block cost and the cluster sweeps
        # on high-priority streams -- the step's critical path -- while
        # row/WTA/LR fill the SMs the clusters leave free, so their event
        # durations include waiting for SMs; D1 runs serially.
        crit = CRITICAL if st.engine == 3 else asd.abi.STAGES
        top = max((k for k in crit if prof[k]["launches"]), key=lambda k: prof[k]["ms"])
        tp = prof[top]
        nl = max(1, tp["launches"])
        avg_ms = tp["ms"] / nl
        alg_b = tp["alg_bytes"] / nl
        alg_o = tp["alg_ops"] / nl
        hbm_ach = alg_b / (avg_ms / 1000.0) / 1e9
        tot_ms = sum(prof[k]["ms"] for k in asd.abi.STAGES)
        stage_share = {k: round(prof[k]["ms"] / max(1e-9, tot_ms), 4) for k in asd.abi.STAGES
                       if prof[k]["launches"]}
        frames_per_launch = st.group if st.engine == 3 else min(args.max_batch, B)
        traffic, step_dram = None, None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        headline = args.config == "C" and args.block == 1 and args.lr_mode == 0 and not args.p2
        if os.path.exists(tpath) and headline:
            try:                      # the ncu capture in the file is of the config-C headline line
                tj = json.load(open(tpath))
                if tj.get(top) is not None:
                    traffic = tj[top] * frames_per_launch
                ks = [k for k in ("census", "down", "up", "row", "wta", "lr") if tj.get(k) is not None]
                step_dram = {"bytes_per_frame": round(sum(tj[k] for k in ks)), "kernels": ks,
                             "survey_8d_algorithmic_bytes_per_frame": [0.26e9, 0.50e9],
                             "ratio_to_8d": [round(sum(tj[k] for k in ks) / 0.50e9, 2),
                                             round(sum(tj[k] for k in ks) / 0.26e9, 2)],
                             "source": "profiles/ncu_traffic.json (ncu dram__bytes_read+write per launch / frames)"}
            except Exception:
                traffic = None
        if alg_o > 0:
            ach = alg_o / (avg_ms / 1000.0) / 1e12
            roof = {"bound": "alu", "achieved": round(ach, 3), "peak": round(alu_peak, 2),
                    "unit": "Tops/s", "frac": round(ach / alu_peak, 4), "traffic": traffic,
                    "alg_ops_per_launch": alg_o,
                    "op_model": "SURVEY §8(d): 5.5 packed lane-ops per cell-path + 2 per cell of Hamming cost",
                    "peak_source": f"{nsm} SMs x 128 int lane-ops/clk x {sm_mhz:.0f} MHz "
                                   "(profiles/r02_ubench.txt: VIMNMX.U16x2 / IADD3 issue 123-128 lane-ops/clk/SM)",
                    "hbm_view": {"achieved": round(hbm_ach, 1), "peak": hbm_peak, "unit": "GB/s",
                                 "frac": round(hbm_ach / hbm_peak, 4)}}
            m = op_models(top, params["paths"], args.block > 1)
            if m:
                roof["frac_minimal_model"] = round(ach / alu_peak * m[1] / m[0], 4)
                roof["minimal_model"] = "DESIGN.md §5: 2.5 lane-ops per cell-path + 3 per cell of cost"
        else:
            roof = {"bound": "hbm", "achieved": round(hbm_ach, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(hbm_ach / hbm_peak, 4), "traffic": traffic,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk else "fallback B200_PROFILING.md"}
        roof.update({"kernel": KERNEL_NAMES[top], "alg_bytes_per_launch": alg_b,
                     "avg_launch_ms": round(avg_ms, 4), "launches": nl, "frames_per_launch": frames_per_launch})
        if step_dram:
            roof["step_dram"] = step_dram
        # share of the profiled pass the critical (sweep) streams are busy
        pipeline = None
        if timeline and st.engine == 3:
            iv = sorted((a, b) for k, a, b in timeline if k in CRITICAL)
            busy, cur0, cur1 = 0.0, None, None
            for a, b in iv:
                if cur1 is None or a > cur1:
                    if cur1 is not None:
                        busy += cur1 - cur0
                    cur0, cur1 = a, b
                else:
                    cur1 = max(cur1, b)
            if cur1 is not None:
                busy += cur1 - cur0
            span = max(b for _, _, b in timeline) - min(a for _, a, _ in timeline)
            pipeline = {"group_frames": st.group, "critical_stages": list(CRITICAL),
                        "critical_stream_busy": round(busy / max(1e-9, span), 4),
                        "profiled_steps": psteps,
                        "note": "stage_ms from a separate profiled pass; row/wta/lr overlap the sweeps"}
        gate = None
        if not args.no_gate and args.block == 1 and args.lr_mode == 0:
            gate = d1_gate(asd, params, L, R, dev, hbm_peak, traffic_ok=args.config == "C")
        line = {
            "metric": METRIC if args.config == "C" else METRIC_D, "value": round(value, 3), "unit": "frames/s",
            "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
            "higher_is_better": True, "scaling": "strong" if args.job else "weak", "vs_baseline": None,
            "dtype": "u16",
            "data": "synthetic",
            "gcells_per_s": round(value * cfg.cells / 1e9, 3),
            "config": bench_config(args, world),
            "run": {"frames_per_step_per_gpu": B, "max_batch": args.max_batch,
                    "distinct_frames": POOL, "engine": st.plan_info},
            "roofline": roof,
            "parity": parity if not args.no_parity else None,
            "stage_ms": {k: round(prof[k]["ms"] / psteps, 3) for k in asd.abi.STAGES if prof[k]["launches"]},
            "stage_share": stage_share,
            "pipeline": pipeline,
            "hbm_gate": gate,
            "clocks": clk.summary(),
            "gpu_launches": lp * args.steps,
            "checksum_frames": int(len(st_all)),
            "checksum0": int(st_all[0, 0]) & 0xFFFFFFFF,
            "valid_frac": round(float(st_all[:, 1].astype(np.int64).sum()) / (len(st_all) * H * W), 4),
        }
        if e2e:
            if parity_e2e is not None and not args.no_parity:
                e2e["parity"] = parity_e2e
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
            try:
                line["context"] = host_context(params, cpu)
            except Exception as exc:             # context only: never fail the line for it
                line["context"] = {"error": str(exc)[:200]}
        print(json.dumps(line), flush=True)
        bad = (0 if args.no_parity else parity["mismatches"] + (parity_e2e["mismatches"] if parity_e2e else 0))
        if bad:
            print(f"PARITY FAILURE: {bad} frame(s) differ from the oracle", file=sys.stderr, flush=True)
    st.close()
    if world > 1:
        dist.destroy_process_group()
    if rank == 0 and not args.no_parity and (parity["mismatches"] or (parity_e2e and parity_e2e["mismatches"])):
        sys.exit(1)


if __name__ == "__main__":
    main()

"""Single-core latency of the CPU oracle per frame for configs A-D (SURVEY §8(d)
"Oracle timing (i)"), on the host it runs on -- test infrastructure timing only,
the oracle as it stands (gcc -O2 -ffp-contract=off, one thread).

    python tools/oracle_latency.py [--configs A,B,C,D] [--out profiles/r01d_oracle_latency.json]
"""
import argparse
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="A,B,C,D")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    oracle.build()
    rows = []
    for name in args.configs.split(","):
        cfg = synth.CONFIGS[name]
        left, right, _ = synth.make_pair(name, 0)
        p = oracle.Params(**cfg.params_dict())
        t0 = time.perf_counter()
        oracle.compute(p, left, right)
        dt = time.perf_counter() - t0
        cells = cfg.width * cfg.height * cfg.num_disp
        rows.append({"config": name, "W": cfg.width, "H": cfg.height, "D": cfg.num_disp, "paths": cfg.paths,
                     "seconds_per_frame": round(dt, 4),
                     "ns_per_cell_path": round(dt / (cells * cfg.paths) * 1e9, 3)})
        print(json.dumps(rows[-1]), flush=True)
    res = {"kind": "oracle single-core latency (one frame, one thread)", "cpu": cpu_model(),
           "cores_visible": len(os.sched_getaffinity(0)), "rows": rows}
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

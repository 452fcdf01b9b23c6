"""Stage-by-stage D3 vs oracle mismatch report (development aid, uses oracle/)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle, synth
from tests.gpu_util import gpu_debug

def report(name, d, L, R, engine=3):
    o = oracle.compute(oracle.Params(**d), L, R, debug=True)
    g = gpu_debug(d, L, R, engine)
    out = [name]
    for k, ok in [("agg", "agg"), ("dstar_l", "dstar_l"), ("dstar_r", "dstar_r"), ("mask", "mask"), ("mask_r", "mask_r")]:
        a = g[k].astype(np.int64); b = o[ok].astype(np.int64)
        bad = a != b
        out.append(f"{k}:{bad.sum()}")
        if bad.any() and k == "agg":
            idx = np.argwhere(bad)[:3]
            for (yy, xx, dd) in idx:
                out.append(f" [{yy},{xx},{dd}] g={a[yy,xx,dd]} o={b[yy,xx,dd]}")
            ys = np.unique(np.argwhere(bad)[:, 0]); xs = np.unique(np.argwhere(bad)[:, 1])
            out.append(f" rows {ys[:5]}..{len(ys)} cols {xs[:5]}..{len(xs)}")
    for k, ok in [("disp_l", "dl"), ("disp_r", "dr")]:
        out.append(f"{k}:{(g[k].view(np.uint32) != o[ok].view(np.uint32)).sum()}")
    print(" ".join(out), flush=True)

cfg = synth.CONFIGS
L, R, _ = synth.make_pair("A", 0); report("A", cfg["A"].params_dict(), L, R)
d = cfg["A"].params_dict(); d.update(paths=8); report("A8", d, L, R)
L, R, _ = synth.make_pair("B", 0); report("B", cfg["B"].params_dict(), L, R)
L, R, _ = synth.make_pair("C", 0); report("C", cfg["C"].params_dict(), L, R)

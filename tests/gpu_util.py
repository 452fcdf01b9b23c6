"""Helpers for the -m gpu parity tests: run the CUDA path through the C ABI
(paper_2201_11924_b200.Stereo) and compare it with the oracle."""
from __future__ import annotations

import numpy as np

import oracle
import paper_2201_11924_b200 as asd


def params_pair(d: dict):
    return asd.Params(**d), oracle.Params(**d)


def gpu_debug(d: dict, left: np.ndarray, right: np.ndarray, engine: int = 0) -> dict:
    """All stage outputs of one frame via asd_depth_debug (engine: 0 auto, 1 D1, 3 D3)."""
    import pytest
    import torch
    p = asd.Params(**d, engine=engine)
    H, W, D = p.height, p.width, p.num_disp
    dev = "cuda"
    sig = torch.int32 if p.nbits <= 32 else torch.int64
    outs = {
        "census_l": torch.empty(H, W, dtype=sig, device=dev),
        "census_r": torch.empty(H, W, dtype=sig, device=dev),
        "cost": torch.empty(H, W, D, dtype=torch.uint8, device=dev),
        "agg": torch.empty(H, W, D, dtype=torch.int16, device=dev),
        "dstar_l": torch.empty(H, W, dtype=torch.int16, device=dev),
        "dstar_r": torch.empty(H, W, dtype=torch.int16, device=dev),
        "disp_l": torch.empty(H, W, dtype=torch.float32, device=dev),
        "disp_r": torch.empty(H, W, dtype=torch.float32, device=dev),
        "mask": torch.empty(H, W, dtype=torch.uint8, device=dev),
        "mask_r": torch.empty(H, W, dtype=torch.uint8, device=dev),
    }
    disp = torch.empty(H, W, dtype=torch.float32, device=dev)
    depth = torch.empty(H, W, dtype=torch.float32, device=dev)
    L = torch.from_numpy(np.ascontiguousarray(left)).to(dev)
    R = torch.from_numpy(np.ascontiguousarray(right)).to(dev)
    try:
        st = asd.Stereo(p, 0, 1)
    except asd.AsdError as e:
        if engine == 3 and e.code == asd.ASD_E_UNSUPPORTED:
            pytest.skip(f"outside the D3 envelope: {e}")
        raise
    with st:
        assert engine == 0 or st.engine == engine
        st.asd_depth_debug(L, R, outs, disp, depth)
        torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in outs.items()}
    g["census_l"] = g["census_l"].view(np.uint32 if p.nbits <= 32 else np.uint64)
    g["census_r"] = g["census_r"].view(np.uint32 if p.nbits <= 32 else np.uint64)
    g["agg"] = g["agg"].view(np.uint16)
    g["disp"] = disp.cpu().numpy()
    g["depth"] = depth.cpu().numpy()
    return g


def assert_bits_equal(a: np.ndarray, b: np.ndarray, what: str):
    a = np.ascontiguousarray(a, np.float32).view(np.uint32)
    b = np.ascontiguousarray(b, np.float32).view(np.uint32)
    bad = a != b
    assert not bad.any(), f"{what}: {bad.sum()} of {bad.size} differ, first at {np.argwhere(bad)[:5].tolist()}"


def assert_equal(a, b, what):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    bad = a != b
    assert not bad.any(), (f"{what}: {bad.sum()} of {bad.size} differ, first at "
                           f"{np.argwhere(bad)[:5].tolist()}: gpu={a[bad][:5]} oracle={b[bad][:5]}")


def assert_depth_close(gz: np.ndarray, oz: np.ndarray, rel: float = 1e-5):
    gn, on = np.isnan(gz), np.isnan(oz)
    assert_equal(gn, on, "depth NaN pattern")
    v = ~on
    if v.any():
        err = np.abs(gz[v].astype(np.float64) - oz[v]) / np.abs(oz[v])
        assert err.max() <= rel, f"depth rel err {err.max():.3g} > {rel}"


def compare_full(g: dict, o: dict, stages=True):
    """GPU debug outputs vs oracle.compute(..., debug=True): bit-exact except depth."""
    if stages:
        assert_equal(g["census_l"].astype(np.uint64), o["census_l"], "census_l")
        assert_equal(g["census_r"].astype(np.uint64), o["census_r"], "census_r")
        assert_equal(g["cost"], o["cost"], "cost")
        assert_equal(g["agg"].astype(np.uint32), o["agg"], "agg")
    assert_equal(g["dstar_l"], o["dstar_l"], "dstar_l")
    assert_equal(g["dstar_r"], o["dstar_r"], "dstar_r")
    assert_equal(g["mask"], o["mask"], "mask")
    assert_equal(g["mask_r"], o["mask_r"], "mask_r")
    assert_bits_equal(g["disp_l"], o["dl"], "dl")
    assert_bits_equal(g["disp_r"], o["dr"], "dr")
    assert_bits_equal(g["disp"], o["disp"], "disp")
    assert_depth_close(g["depth"], o["depth"])


def oracle_frames(d: dict, Ls, Rs, threads: int = 0) -> list:
    """oracle.compute on every frame, one frame per host thread (ctypes releases
    the GIL), memory-bounded (about 1.6 GB per config-C frame)."""
    import os
    import threading
    p = oracle.Params(**{k: v for k, v in d.items() if k != "engine"})
    oracle.lib()
    n = len(Ls)
    if threads <= 0:
        try:
            import psutil
            mem = int(psutil.virtual_memory().available // (2.0 * 1.6e9 * max(1, p.width * p.height * p.num_disp / 117964800)))
        except Exception:
            mem = 4
        threads = max(1, min(n, len(os.sched_getaffinity(0)), mem, 16))
    out = [None] * n
    for k in range(0, n, threads):
        part = list(range(k, min(n, k + threads)))

        def run(i):
            out[i] = oracle.compute(p, Ls[i], Rs[i])

        ths = [threading.Thread(target=run, args=(i,)) for i in part]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
    return out


def oracle_sig(o) -> tuple:
    """(checksum, valid count) of an oracle frame (asd_frame_stats fields)."""
    return oracle.checksum(o["dstar_l"], o["mask"]), int((o["mask"] == 0).sum())

"""CPU oracle for the active-stereo depth path of arXiv 2201.11924 (TEST INFRASTRUCTURE).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2201_11924_b200`` never imports it, and the two share no code.

The arithmetic lives in ``asd_oracle.c`` (plain scalar C99, gcc -O2
-ffp-contract=off); this module only marshals numpy arrays through ctypes.
Each wrapper names the PAPER.md / SPEC.md passage its C function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "asd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

MASK_BORDER, MASK_UNIQUE, MASK_LR, MASK_NONPOS = 1, 2, 4, 8


def build(force: bool = False) -> str:
    """Compile asd_oracle.c -> liboracle.so (gcc, -O2 -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class OracleParams(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("min_disp", ctypes.c_int32), ("num_disp", ctypes.c_int32),
                ("census_w", ctypes.c_int32), ("census_h", ctypes.c_int32),
                ("p1", ctypes.c_int32), ("p2", ctypes.c_int32),
                ("paths", ctypes.c_int32), ("uniqueness", ctypes.c_int32),
                ("lr_max_diff", ctypes.c_float), ("subpixel", ctypes.c_int32),
                ("focal_px", ctypes.c_float), ("baseline_m", ctypes.c_float),
                ("block_w", ctypes.c_int32), ("block_h", ctypes.c_int32),
                ("median_ksize", ctypes.c_int32), ("lr_mode", ctypes.c_int32)]


@dataclass
class Params:
    """Stereo configuration (SPEC S:257-260 StereoConfig; defaults)."""
    width: int
    height: int
    num_disp: int = 64
    min_disp: int = 0
    census_w: int = 9
    census_h: int = 7
    p1: int = 8
    p2: int = 32
    paths: int = 4
    uniqueness: int = 10
    lr_max_diff: float = 1.0
    subpixel: int = 1
    focal_px: float = 430.0
    baseline_m: float = 0.055
    block_w: int = 1          # SGBM block; 1 x 1 = plain SGM
    block_h: int = 1
    median_ksize: int = 0     # 0 (off), 3, 5
    lr_mode: int = 0          # right view: 0 = R1 (re-index, c10), 1 = R2 (own SGM, c24)

    @property
    def nbits(self) -> int:
        return (self.census_w * self.census_h) // 2

    def c(self) -> OracleParams:
        return OracleParams(self.width, self.height, self.min_disp, self.num_disp,
                            self.census_w, self.census_h, self.p1, self.p2, self.paths,
                            self.uniqueness, self.lr_max_diff, self.subpixel,
                            self.focal_px, self.baseline_m, self.block_w, self.block_h,
                            self.median_ksize, self.lr_mode)


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_checksum.restype = ctypes.c_uint32
        _lib.oracle_compute.restype = ctypes.c_int
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def census(p: Params, img: np.ndarray) -> np.ndarray:
    """O1 -- CSCT.  img u8[H][W] -> u64[H][W]."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    out = np.empty((p.height, p.width), np.uint64)
    lib().oracle_census(ctypes.byref(p.c()), _p(img), _p(out))
    return out


def cost(p: Params, cl: np.ndarray, cr: np.ndarray) -> np.ndarray:
    """O2 -- Hamming matching cost.  -> u8[H][W][D]."""
    cl = np.ascontiguousarray(cl, np.uint64)
    cr = np.ascontiguousarray(cr, np.uint64)
    out = np.empty((p.height, p.width, p.num_disp), np.uint8)
    lib().oracle_cost(ctypes.byref(p.c()), _p(cl), _p(cr), _p(out))
    return out


def cost_right(p: Params, cl: np.ndarray, cr: np.ndarray) -> np.ndarray:
    """O2 with the right view as reference (reading c24).  -> u8[H][W][D]."""
    cl = np.ascontiguousarray(cl, np.uint64)
    cr = np.ascontiguousarray(cr, np.uint64)
    out = np.empty((p.height, p.width, p.num_disp), np.uint8)
    lib().oracle_cost_right(ctypes.byref(p.c()), _p(cl), _p(cr), _p(out))
    return out


def block_cost(p: Params, C: np.ndarray) -> np.ndarray:
    """O2b -- SGBM block cost (reading c19).  C u8[H][W][D] -> u32[H][W][D]."""
    C = np.ascontiguousarray(C, np.uint8)
    out = np.empty((p.height, p.width, p.num_disp), np.uint32)
    lib().oracle_block_cost(ctypes.byref(p.c()), _p(C), _p(out))
    return out


def sgm32(p: Params, C: np.ndarray) -> np.ndarray:
    """O3 on a u32 cost volume (SGBM block costs).  -> u32[H][W][D]."""
    C = np.ascontiguousarray(C, np.uint32)
    out = np.empty((p.height, p.width, p.num_disp), np.uint32)
    lib().oracle_sgm32(ctypes.byref(p.c()), _p(C), _p(out))
    return out


def chain(C: np.ndarray, p1: int, p2: int) -> np.ndarray:
    """O3 recursion along one line.  C[n][D] -> L[n][D] (u32)."""
    C = np.ascontiguousarray(C, np.uint32)
    n, D = C.shape
    out = np.empty((n, D), np.uint32)
    lib().oracle_chain(n, D, p1, p2, _p(C), _p(out))
    return out


def directions(paths: int):
    out = []
    for i in range(paths):
        rx, ry = ctypes.c_int(), ctypes.c_int()
        lib().oracle_dir(i, ctypes.byref(rx), ctypes.byref(ry))
        out.append((rx.value, ry.value))
    return out


def sgm_path(p: Params, C: np.ndarray, rx: int, ry: int) -> np.ndarray:
    """L_r for one direction r."""
    C = np.ascontiguousarray(C, np.uint8)
    out = np.empty((p.height, p.width, p.num_disp), np.uint32)
    lib().oracle_sgm_path(ctypes.byref(p.c()), _p(C), rx, ry, _p(out))
    return out


def sgm(p: Params, C: np.ndarray) -> np.ndarray:
    """O3 -- S = sum_r L_r.  -> u32[H][W][D]."""
    C = np.ascontiguousarray(C, np.uint8)
    out = np.empty((p.height, p.width, p.num_disp), np.uint32)
    lib().oracle_sgm(ctypes.byref(p.c()), _p(C), _p(out))
    return out


def sgm_pixel(p: Params, cl: np.ndarray, cr: np.ndarray, x: int, y: int) -> np.ndarray:
    """S(x,y,.) for one pixel from the census images (walks each path's line)."""
    cl = np.ascontiguousarray(cl, np.uint64)
    cr = np.ascontiguousarray(cr, np.uint64)
    out = np.empty(p.num_disp, np.uint32)
    lib().oracle_sgm_pixel_from_census(ctypes.byref(p.c()), _p(cl), _p(cr), x, y, _p(out))
    return out


def wta_left(p: Params, S: np.ndarray):
    """O4+O5 left view.  -> (dstar i16, mask u8, dl f32)."""
    S = np.ascontiguousarray(S, np.uint32)
    ds = np.empty((p.height, p.width), np.int16)
    m = np.empty((p.height, p.width), np.uint8)
    dl = np.empty((p.height, p.width), np.float32)
    lib().oracle_wta_left(ctypes.byref(p.c()), _p(S), _p(ds), _p(m), _p(dl))
    return ds, m, dl


def wta_right(p: Params, S: np.ndarray):
    """O6 right view by re-indexing S (reading c10)."""
    S = np.ascontiguousarray(S, np.uint32)
    ds = np.empty((p.height, p.width), np.int16)
    m = np.empty((p.height, p.width), np.uint8)
    dr = np.empty((p.height, p.width), np.float32)
    lib().oracle_wta_right(ctypes.byref(p.c()), _p(S), _p(ds), _p(m), _p(dr))
    return ds, m, dr


def lr_depth(p: Params, dl, dr, mask_r, mask):
    """O7+O8.  mask is updated in a copy; -> (mask, disp f32, depth f64)."""
    dl = np.ascontiguousarray(dl, np.float32)
    dr = np.ascontiguousarray(dr, np.float32)
    mask_r = np.ascontiguousarray(mask_r, np.uint8)
    m = np.array(mask, dtype=np.uint8, copy=True, order="C")
    disp = np.empty((p.height, p.width), np.float32)
    z = np.empty((p.height, p.width), np.float64)
    lib().oracle_lr_depth(ctypes.byref(p.c()), _p(dl), _p(dr), _p(mask_r), _p(m), _p(disp), _p(z))
    return m, disp, z


def median(p: Params, dl: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """O9 -- lower median over the valid k x k neighbours (reading c20)."""
    dl = np.ascontiguousarray(dl, np.float32)
    mask = np.ascontiguousarray(mask, np.uint8)
    out = np.empty_like(dl)
    lib().oracle_median(ctypes.byref(p.c()), _p(dl), _p(mask), _p(out))
    return out


class OracleCamera(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("fx", ctypes.c_float), ("fy", ctypes.c_float),
                ("cx", ctypes.c_float), ("cy", ctypes.c_float)]


def register(ir: tuple, rgb: tuple, R, t, z: np.ndarray) -> np.ndarray:
    """O10 -- depth registration into the RGB frame (reading c21).
    ir / rgb = (width, height, fx, fy, cx, cy); R 3x3, t 3; z f32[H_ir][W_ir]
    (NaN = invalid) -> f32[H_rgb][W_rgb] (NaN = no sample)."""
    z = np.ascontiguousarray(z, np.float32)
    R = np.ascontiguousarray(np.asarray(R, np.float32).reshape(9))
    t = np.ascontiguousarray(np.asarray(t, np.float32).reshape(3))
    ci, cr = OracleCamera(*ir), OracleCamera(*rgb)
    out = np.empty((rgb[1], rgb[0]), np.float32)
    lib().oracle_register(ctypes.byref(ci), ctypes.byref(cr), _p(R), _p(t), _p(z), _p(out))
    return out


def checksum(dstar: np.ndarray, mask: np.ndarray) -> int:
    """Per-frame checksum of (d*, mask)."""
    dstar = np.ascontiguousarray(dstar, np.int16)
    mask = np.ascontiguousarray(mask, np.uint8)
    return int(lib().oracle_checksum(dstar.size, _p(dstar), _p(mask)))


def compute(p: Params, left: np.ndarray, right: np.ndarray, debug: bool = False) -> dict:
    """The whole path O1..O8 (S:366-368 compute_depth; P:289 stage order)."""
    left = np.ascontiguousarray(left, np.uint8)
    right = np.ascontiguousarray(right, np.uint8)
    H, W, D = p.height, p.width, p.num_disp
    out = {"disp": np.empty((H, W), np.float32), "depth": np.empty((H, W), np.float64),
           "dstar_l": np.empty((H, W), np.int16), "dstar_r": np.empty((H, W), np.int16),
           "dl": np.empty((H, W), np.float32), "dr": np.empty((H, W), np.float32),
           "mask": np.empty((H, W), np.uint8), "mask_r": np.empty((H, W), np.uint8)}
    if debug:
        out.update({"census_l": np.empty((H, W), np.uint64), "census_r": np.empty((H, W), np.uint64),
                    "cost": np.empty((H, W, D), np.uint8), "agg": np.empty((H, W, D), np.uint32)})
    g = lambda k: _p(out[k]) if k in out else None  # noqa: E731
    rc = lib().oracle_compute(ctypes.byref(p.c()), _p(left), _p(right), g("disp"), g("depth"),
                              g("census_l"), g("census_r"), g("cost"), g("agg"),
                              g("dstar_l"), g("dstar_r"), g("dl"), g("dr"), g("mask"), g("mask_r"))
    if rc != 0:
        raise MemoryError("oracle_compute: allocation failed")
    return out


# ------------------------------------------------------------------ O0 noise
class OracleNoise(ctypes.Structure):
    _fields_ = [("k", ctypes.c_double), ("theta", ctypes.c_double), ("mu", ctypes.c_double),
                ("sigma", ctypes.c_double), ("scale", ctypes.c_double)]


D415_NOISE = dict(k=3.98, theta=0.254, mu=-0.231, sigma=0.83, scale=1.0)


def philox(ctr, key):
    """Philox4x32-10 of one 128-bit counter under a 64-bit key (4 x u32 out)."""
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().oracle_philox4x32_10(c, k, o)
    return list(o)


def sensor_noise(clean: np.ndarray, seed: int, frame0: int = 0, view: int = 0, f64: bool = False, **noise):
    """O0 -- gamma*I + n, quantised to u8 (readings c17, c22).
    clean [n][H][W] or [H][W] (DN units) -> u8 of the same shape (and the
    unrounded values when f64)."""
    q = dict(D415_NOISE); q.update(noise)
    c = np.ascontiguousarray(clean, np.float64)
    shp = c.shape
    c3 = c.reshape((-1,) + shp[-2:])
    out = np.empty(c3.shape, np.uint8)
    val = np.empty(c3.shape, np.float64) if f64 else None
    lib().oracle_sensor_noise(ctypes.byref(OracleNoise(**q)), ctypes.c_uint64(seed), c3.shape[0],
                              shp[-1], shp[-2], ctypes.c_uint32(frame0), ctypes.c_uint32(view),
                              _p(c3), _p(out), _p(val) if f64 else None)
    return (out.reshape(shp), val.reshape(shp)) if f64 else out.reshape(shp)


def noise_samples(n: int, seed: int, frame: int = 0, view: int = 0, **noise):
    """(gamma, n) samples of pixels 0..n-1 of one stream (before the scale blend)."""
    q = dict(D415_NOISE); q.update(noise)
    g = np.empty(n, np.float64)
    a = np.empty(n, np.float64)
    lib().oracle_noise_samples(ctypes.byref(OracleNoise(**q)), ctypes.c_uint64(seed), n,
                               ctypes.c_uint32(frame), ctypes.c_uint32(view), _p(g), _p(a))
    return g, a


def rectify(Hm, img: np.ndarray) -> np.ndarray:
    """O00 -- homography warp with bilinear sampling (reading c23).
    Hm maps output pixel coordinates to input coordinates."""
    img = np.ascontiguousarray(img, np.uint8)
    Hd = np.ascontiguousarray(np.asarray(Hm, np.float64).reshape(9))
    out = np.empty_like(img)
    rc = lib().oracle_rectify(_p(Hd), img.shape[1], img.shape[0], _p(img), _p(out))
    if rc != 0:
        raise ValueError("singular homography")
    return out

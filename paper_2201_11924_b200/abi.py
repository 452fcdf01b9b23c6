"""Thin ctypes binding of libasd.so (include/asd.h).  Argument marshalling only:
every step of the depth path runs in the library's sm_100a kernels.

Names mirror the C ABI: ``asd_create`` / ``asd_depth`` / ``asd_depth_batch`` /
``asd_depth_batch_host`` / ``asd_depth_debug`` / ``asd_destroy`` are wrapped by
:class:`Stereo`.  Tensors are passed as raw pointers (``tensor.data_ptr()``)
together with torch's current CUDA stream; this module never computes anything
itself, and it raises if the library is missing (there is no fallback path).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_PKG = os.path.dirname(os.path.abspath(__file__))
# ASD_LIB overrides the library path (A/B timing of kernel variants, tools/)
LIB_PATH = os.environ.get("ASD_LIB") or os.path.join(_PKG, "lib", "libasd.so")

ASD_OK, ASD_E_INVALID_ARG, ASD_E_UNSUPPORTED, ASD_E_CUDA, ASD_E_OOM = 0, -1, -2, -3, -4
MASK_BORDER, MASK_UNIQUE, MASK_LR, MASK_NONPOS = 1, 2, 4, 8


class AsdError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"asd error {code}: {msg}")
        self.code = code


class asd_params(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("min_disp", ctypes.c_int32), ("num_disp", ctypes.c_int32),
                ("census_w", ctypes.c_int32), ("census_h", ctypes.c_int32),
                ("p1", ctypes.c_int32), ("p2", ctypes.c_int32),
                ("paths", ctypes.c_int32), ("uniqueness", ctypes.c_int32),
                ("lr_max_diff", ctypes.c_float), ("subpixel", ctypes.c_int32),
                ("focal_px", ctypes.c_float), ("baseline_m", ctypes.c_float),
                ("engine", ctypes.c_int32),
                ("block_w", ctypes.c_int32), ("block_h", ctypes.c_int32),
                ("median_ksize", ctypes.c_int32), ("lr_mode", ctypes.c_int32)]


class asd_frame_stats(ctypes.Structure):
    _fields_ = [("checksum", ctypes.c_uint32), ("valid", ctypes.c_uint32),
                ("depth_sum", ctypes.c_float), ("reserved", ctypes.c_uint32)]


class asd_debug_out(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("census_l", "census_r", "cost", "agg", "dstar_l", "dstar_r",
                 "disp_l", "disp_r", "mask", "mask_r")]


STAGES = ("census", "dir", "wta", "lr", "down", "up", "row", "block")


class asd_stage_times(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 8), ("alg_bytes", ctypes.c_double * 8),
                ("alg_ops", ctypes.c_double * 8),
                ("launches", ctypes.c_int32 * 8), ("dropped", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


# (name, restype, argtypes) of every exported symbol declared in include/asd.h
_VP, _I, _SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
SYMBOLS = [
    ("asd_version", _I, []),
    ("asd_scratch_bytes", _SZ, [ctypes.POINTER(asd_params), _I]),
    ("asd_create", _I, [ctypes.POINTER(asd_params), _I, _I, ctypes.POINTER(_VP)]),
    ("asd_destroy", None, [_VP]),
    ("asd_depth", _I, [_VP, _VP, _VP, _VP, _VP, _VP]),
    ("asd_depth_batch", _I, [_VP, _I, _VP, _VP, _VP, _VP, _VP, _VP]),
    ("asd_depth_batch_host", _I, [_VP, _I, _VP, _VP, _VP, _VP, _VP, _VP]),
    ("asd_depth_debug", _I, [_VP, _VP, _VP, ctypes.POINTER(asd_debug_out), _VP, _VP, _VP]),
    ("asd_launches_per_batch", _I, [_VP, _I]),
    ("asd_set_group", _I, [_VP, _I]),
    ("asd_group", _I, [_VP]),
    ("asd_engine", _I, [_VP]),
    ("asd_frames_per_wave", _I, [_VP]),
    ("asd_plan_info", _I, [_VP, ctypes.c_char_p, _I]),
    ("asd_profile_begin", _I, [_VP, _I]),
    ("asd_profile_end", _I, [_VP, ctypes.POINTER(asd_stage_times)]),
    ("asd_profile_timeline", _I, [_VP, _I, ctypes.POINTER(ctypes.c_int32),
                                  ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]),
    ("asd_register_depth", _I, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                _I, _VP, _VP, _VP]),
    ("asd_sensor_noise", _I, [ctypes.c_void_p, ctypes.c_uint64, _I, _I, _I, ctypes.c_uint32,
                              ctypes.c_uint32, _VP, _VP, _VP]),
    ("asd_rectify", _I, [ctypes.c_void_p, _I, _I, _I, _VP, _VP, _VP]),
    ("asd_strerror", ctypes.c_char_p, [_I]),
    ("asd_last_error", ctypes.c_char_p, [_VP]),
]

_lib = None


def load(path: str = LIB_PATH):
    """Load libasd.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"{path} not found: build it with "
                              "`python -m paper_2201_11924_b200.build` (no CPU fallback exists)")
        lib = ctypes.CDLL(path)
        for name, res, args in SYMBOLS:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


@dataclass
class Params:
    """asd_params (include/asd.h; fields of SPEC S:257-260 StereoConfig).

    The defaults are this repo's config-C defaults (8 paths, median off), not
    SPEC S:388's (4 paths, median 3).  p1 / p2 left as None follow S:388 scaled
    by the block area: P1 = 8 * bw * bh, P2 = 32 * bw * bh (8 / 32 for SGM)."""
    width: int
    height: int
    num_disp: int = 64
    min_disp: int = 0
    census_w: int = 9
    census_h: int = 7
    p1: int | None = None
    p2: int | None = None
    paths: int = 8
    uniqueness: int = 10
    lr_max_diff: float = 1.0
    subpixel: int = 1
    focal_px: float = 430.0
    baseline_m: float = 0.055
    engine: int = 0            # ASD_ENGINE_AUTO (0), _D1 (1), _D3 (3)
    block_w: int = 1           # SGBM block (reading c19); 1 x 1 = SGM
    block_h: int = 1
    median_ksize: int = 0      # 0 / 3 / 5 (reading c20)
    lr_mode: int = 0           # right view: 0 = R1 re-index (c10), 1 = R2 own SGM (c24)

    def __post_init__(self):
        area = max(1, self.block_w) * max(1, self.block_h)
        if self.p1 is None:
            self.p1 = 8 * area
        if self.p2 is None:
            self.p2 = 32 * area

    def c(self) -> asd_params:
        return asd_params(self.width, self.height, self.min_disp, self.num_disp, self.census_w,
                          self.census_h, self.p1, self.p2, self.paths, self.uniqueness,
                          self.lr_max_diff, self.subpixel, self.focal_px, self.baseline_m,
                          self.engine, self.block_w, self.block_h, self.median_ksize, self.lr_mode)

    @property
    def nbits(self) -> int:
        return (self.census_w * self.census_h) // 2


def _check(rc: int, ctx=None):
    if rc != ASD_OK:
        lib = load()
        msg = lib.asd_last_error(ctx).decode() if ctx is not None else lib.asd_last_error(None).decode()
        raise AsdError(rc, f"{lib.asd_strerror(rc).decode()}: {msg}")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class asd_camera(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("fx", ctypes.c_float), ("fy", ctypes.c_float),
                ("cx", ctypes.c_float), ("cy", ctypes.c_float)]


def register_depth(ir: tuple, rgb: tuple, R, t, depth, out=None, stream=None):
    """asd_register_depth: depth maps (torch f32 CUDA, [n][H][W] or [H][W], NaN =
    invalid) into the RGB frame.  ir / rgb = (width, height, fx, fy, cx, cy);
    R 3x3, t 3 (IR -> RGB coordinates).  Returns out [n][H_rgb][W_rgb]."""
    import torch
    squeeze = depth.dim() == 2
    d = depth.unsqueeze(0) if squeeze else depth
    assert d.is_cuda and d.dtype == torch.float32 and d.is_contiguous()
    n = d.shape[0]
    if out is None:
        out = torch.empty(n, rgb[1], rgb[0], device=d.device, dtype=torch.float32)
    Rc = (ctypes.c_float * 9)(*[float(v) for v in list(__import__("numpy").asarray(R, "float32").reshape(9))])
    tc = (ctypes.c_float * 3)(*[float(v) for v in list(__import__("numpy").asarray(t, "float32").reshape(3))])
    ci, cr = asd_camera(*ir), asd_camera(*rgb)
    _check(load().asd_register_depth(ctypes.byref(ci), ctypes.byref(cr), Rc, tc, n, _ptr(d), _ptr(out),
                                     _stream(stream)))
    return out[0] if squeeze else out


class asd_noise(ctypes.Structure):
    _fields_ = [("k", ctypes.c_double), ("theta", ctypes.c_double), ("mu", ctypes.c_double),
                ("sigma", ctypes.c_double), ("scale", ctypes.c_double)]


D415_NOISE = dict(k=3.98, theta=0.254, mu=-0.231, sigma=0.83, scale=1.0)


def sensor_noise(clean, seed: int, frame0: int = 0, view: int = 0, out=None, stream=None, **noise):
    """asd_sensor_noise: clean IR intensities (torch f32 CUDA, [n][H][W] or
    [H][W], DN units) -> u8 noisy images (readings c17, c22)."""
    import torch
    q = dict(D415_NOISE); q.update(noise)
    squeeze = clean.dim() == 2
    c = clean.unsqueeze(0) if squeeze else clean
    assert c.is_cuda and c.dtype == torch.float32 and c.is_contiguous()
    n, H, W = c.shape
    if out is None:
        out = torch.empty(n, H, W, device=c.device, dtype=torch.uint8)
    _check(load().asd_sensor_noise(ctypes.byref(asd_noise(**q)), ctypes.c_uint64(seed), n, W, H,
                                   ctypes.c_uint32(frame0), ctypes.c_uint32(view), _ptr(c), _ptr(out),
                                   _stream(stream)))
    return out[0] if squeeze else out


def rectify(Hm, images, out=None, stream=None):
    """asd_rectify: warp u8 images (torch CUDA, [n][H][W] or [H][W]) by the
    homography Hm (output -> input pixel coordinates; reading c23)."""
    import torch
    squeeze = images.dim() == 2
    im = images.unsqueeze(0) if squeeze else images
    assert im.is_cuda and im.dtype == torch.uint8 and im.is_contiguous()
    n, H, W = im.shape
    if out is None:
        out = torch.empty_like(im)
    Hd = (ctypes.c_double * 9)(*[float(v) for v in __import__("numpy").asarray(Hm, "float64").reshape(9)])
    _check(load().asd_rectify(Hd, n, W, H, _ptr(im), _ptr(out), _stream(stream)))
    return out[0] if squeeze else out


def scratch_bytes(params: Params, max_batch: int = 1) -> int:
    return int(load().asd_scratch_bytes(ctypes.byref(params.c()), max_batch))


class Stereo:
    """One libasd context (asd_create ... asd_destroy) bound to a CUDA device."""

    def __init__(self, params: Params, device: int = 0, max_batch: int = 1):
        self.params = params
        self.device = device
        self.max_batch = max_batch
        self._lib = load()
        ctx = ctypes.c_void_p()
        _check(self._lib.asd_create(ctypes.byref(params.c()), device, max_batch, ctypes.byref(ctx)))
        self._ctx = ctx

    def close(self):
        if getattr(self, "_ctx", None) is not None and self._ctx.value:
            self._lib.asd_destroy(self._ctx)
        self._ctx = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- argument checks (the C ABI takes raw pointers: shapes, dtypes,
    # contiguity and placement are verified here, before any pointer leaves) ----
    def _io(self, host: bool, batch: bool, left, right, out_disp, out_depth, stats=None) -> int:
        import torch
        H, W = self.params.height, self.params.width
        lead = (left.shape[0],) if batch else ()
        if batch and left.dim() != 3:
            raise ValueError(f"left must be [n][{H}][{W}], got {tuple(left.shape)}")
        n = left.shape[0] if batch else 1

        def chk(t, name, dtype, shape):
            if t is None:
                return
            if t.dtype != dtype:
                raise TypeError(f"{name}: dtype {t.dtype}, expected {dtype}")
            if tuple(t.shape) != shape:
                raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {shape}")
            if not t.is_contiguous():
                raise ValueError(f"{name} must be contiguous")
            if host:
                if t.is_cuda:
                    raise ValueError(f"{name} must be a host (CPU, ideally pinned) tensor")
            elif not (t.is_cuda and t.device.index == self.device):
                raise ValueError(f"{name} must be on cuda:{self.device}, got {t.device}")

        chk(left, "left", torch.uint8, lead + (H, W))
        chk(right, "right", torch.uint8, lead + (H, W))
        chk(out_disp, "out_disp", torch.float32, lead + (H, W))
        chk(out_depth, "out_depth", torch.float32, lead + (H, W))
        chk(stats, "stats", torch.int32, (n, 4))
        return n

    # ---- device entry points (torch CUDA tensors) ----
    def asd_depth(self, left, right, out_disp=None, out_depth=None, stream=None):
        self._io(False, False, left, right, out_disp, out_depth)
        _check(self._lib.asd_depth(self._ctx, _ptr(left), _ptr(right), _ptr(out_disp),
                                   _ptr(out_depth), _stream(stream)), self._ctx)

    def asd_depth_batch(self, left, right, out_disp=None, out_depth=None, stats=None, stream=None):
        n = self._io(False, True, left, right, out_disp, out_depth, stats)
        _check(self._lib.asd_depth_batch(self._ctx, n, _ptr(left), _ptr(right), _ptr(out_disp),
                                         _ptr(out_depth), _ptr(stats), _stream(stream)), self._ctx)

    def asd_depth_debug(self, left, right, outs: dict, out_disp=None, out_depth=None, stream=None):
        self._io(False, False, left, right, out_disp, out_depth)
        for k, v in outs.items():
            if v is not None and not (v.is_cuda and v.is_contiguous()):
                raise ValueError(f"debug output {k} must be a contiguous CUDA tensor")
        d = asd_debug_out(**{k: (v.data_ptr() if v is not None else None) for k, v in outs.items()})
        _check(self._lib.asd_depth_debug(self._ctx, _ptr(left), _ptr(right), ctypes.byref(d),
                                         _ptr(out_disp), _ptr(out_depth), _stream(stream)), self._ctx)

    # ---- host entry point (CPU tensors, ideally pinned) ----
    def asd_depth_batch_host(self, left, right, out_disp=None, out_depth=None, stats=None, stream=None):
        n = self._io(True, True, left, right, out_disp, out_depth, stats)
        _check(self._lib.asd_depth_batch_host(self._ctx, n, _ptr(left), _ptr(right), _ptr(out_disp),
                                              _ptr(out_depth), _ptr(stats), _stream(stream)), self._ctx)

    def profile_begin(self, max_launches: int = 65536):
        _check(self._lib.asd_profile_begin(self._ctx, max_launches), self._ctx)

    def profile_end(self) -> dict:
        t = asd_stage_times()
        _check(self._lib.asd_profile_end(self._ctx, ctypes.byref(t)), self._ctx)
        return {name: {"ms": t.ms[i], "alg_bytes": t.alg_bytes[i], "alg_ops": t.alg_ops[i],
                       "launches": t.launches[i]}
                for i, name in enumerate(STAGES)} | {"dropped": t.dropped}

    def profile_timeline(self, max_launches: int = 65536) -> list:
        """[(stage name, start ms, end ms)] per launch since profile_begin, in
        enqueue order (call before profile_end)."""
        st = (ctypes.c_int32 * max_launches)()
        a = (ctypes.c_float * max_launches)()
        b = (ctypes.c_float * max_launches)()
        k = self._lib.asd_profile_timeline(self._ctx, max_launches, st, a, b)
        _check(min(k, 0), self._ctx)
        return [(STAGES[st[i]], a[i], b[i]) for i in range(k)]

    @property
    def group(self) -> int:
        """Frames per D3 pipeline group (asd_set_group)."""
        return int(self._lib.asd_group(self._ctx))

    @group.setter
    def group(self, g: int):
        _check(self._lib.asd_set_group(self._ctx, int(g)), self._ctx)

    @property
    def engine(self) -> int:
        return int(self._lib.asd_engine(self._ctx))

    @property
    def frames_per_wave(self) -> int:
        return int(self._lib.asd_frames_per_wave(self._ctx))

    @property
    def plan_info(self) -> str:
        buf = ctypes.create_string_buffer(512)
        self._lib.asd_plan_info(self._ctx, buf, 512)
        return buf.value.decode()

    def launches_per_batch(self, n: int) -> int:
        return int(self._lib.asd_launches_per_batch(self._ctx, n))

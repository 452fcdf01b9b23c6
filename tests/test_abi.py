"""The C-ABI library loads and exports every symbol include/asd.h declares;
host-side validation works without a GPU (no compute calls here)."""
import ctypes
import os
import re

import pytest

import paper_2201_11924_b200 as asd
from paper_2201_11924_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2201_11924_b200 import build
    build.build()
    return asd.load()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "asd.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(asd_[a-z_]+)\s*\(", hdr)))


def test_exports_every_declared_symbol(lib):
    names = declared_symbols()
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(n for n, _, _ in abi.SYMBOLS) == names
    out = os.popen(f"nm -D --defined-only {abi.LIB_PATH}").read()
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_version_and_strerror(lib):
    assert lib.asd_version() == 3
    assert lib.asd_strerror(0) == b"ok"
    assert lib.asd_strerror(-2) == b"unsupported configuration"


def test_sm100a_only_cubin():
    out = os.popen(f"cuobjdump --list-elf {abi.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


@pytest.mark.parametrize("kw,code", [
    (dict(num_disp=100), asd.ASD_E_UNSUPPORTED),
    (dict(num_disp=512), asd.ASD_E_UNSUPPORTED),
    (dict(census_w=8), asd.ASD_E_INVALID_ARG),
    (dict(census_w=13, census_h=11), asd.ASD_E_UNSUPPORTED),      # nb = 71 > 64
    (dict(p1=10, p2=5), asd.ASD_E_INVALID_ARG),
    (dict(p2=250), asd.ASD_E_UNSUPPORTED),                       # nb + p2 > 255
    (dict(paths=6), asd.ASD_E_INVALID_ARG),
    (dict(min_disp=-1), asd.ASD_E_INVALID_ARG),
    (dict(focal_px=0.0), asd.ASD_E_INVALID_ARG),
    (dict(lr_max_diff=float("nan")), asd.ASD_E_INVALID_ARG),
    (dict(width=3), asd.ASD_E_INVALID_ARG),
    (dict(block_w=2), asd.ASD_E_INVALID_ARG),                    # SGBM block must be odd
    (dict(block_h=17), asd.ASD_E_INVALID_ARG),                   # <= 15
    (dict(block_w=15, block_h=15, p2=6000), asd.ASD_E_UNSUPPORTED),  # 8*(225*12+p2) > 65535
    (dict(median_ksize=4), asd.ASD_E_INVALID_ARG),               # 0, 3 or 5
])
def test_validation(lib, kw, code):
    d = dict(width=64, height=48, num_disp=16, census_w=5, census_h=5)
    d.update(kw)
    p = asd.Params(**d)
    ctx = ctypes.c_void_p()
    assert lib.asd_create(ctypes.byref(p.c()), 0, 1, ctypes.byref(ctx)) == code
    assert not ctx.value
    assert lib.asd_last_error(None)
    assert lib.asd_scratch_bytes(ctypes.byref(p.c()), 1) == 0


def test_scratch_bytes(lib):
    p = asd.Params(1280, 720, 128)
    one = lib.asd_scratch_bytes(ctypes.byref(p.c()), 1)
    assert one >= 1280 * 720 * 128 * 2
    assert lib.asd_scratch_bytes(ctypes.byref(p.c()), 4) >= 4 * 1280 * 720 * 128 * 2
    assert lib.asd_scratch_bytes(ctypes.byref(p.c()), 0) == 0


def test_null_ctx_rejected(lib):
    assert lib.asd_depth(None, None, None, None, None, None) == asd.ASD_E_INVALID_ARG
    assert lib.asd_depth_batch(None, 1, None, None, None, None, None, None) == asd.ASD_E_INVALID_ARG


def test_register_depth_validation(lib):
    """asd_register_depth rejects NULL / out-of-range arguments before touching the GPU."""
    ir = abi.asd_camera(40, 30, 100.0, 100.0, 19.5, 14.5)
    bad = abi.asd_camera(0, 30, 100.0, 100.0, 19.5, 14.5)
    R = (ctypes.c_float * 9)(1, 0, 0, 0, 1, 0, 0, 0, 1)
    t = (ctypes.c_float * 3)(0, 0, 0)
    reg = lib.asd_register_depth
    assert reg(None, ctypes.byref(ir), R, t, 1, None, None, None) == asd.ASD_E_INVALID_ARG
    assert reg(ctypes.byref(ir), ctypes.byref(ir), R, t, -1, None, None, None) == asd.ASD_E_INVALID_ARG
    assert reg(ctypes.byref(ir), ctypes.byref(bad), R, t, 0, None, None, None) == asd.ASD_E_INVALID_ARG
    Rn = (ctypes.c_float * 9)(float("nan"), 0, 0, 0, 1, 0, 0, 0, 1)
    assert reg(ctypes.byref(ir), ctypes.byref(ir), Rn, t, 0, None, None, None) == asd.ASD_E_INVALID_ARG
    assert reg(ctypes.byref(ir), ctypes.byref(ir), R, t, 0, None, None, None) == asd.ASD_OK


def test_sensor_noise_validation(lib):
    q = abi.asd_noise(3.98, 0.254, -0.231, 0.83, 1.0)
    bad = abi.asd_noise(-1.0, 0.254, -0.231, 0.83, 1.0)
    f = lib.asd_sensor_noise
    assert f(None, 1, 1, 8, 8, 0, 0, None, None, None) == asd.ASD_E_INVALID_ARG
    assert f(ctypes.byref(q), 1, -1, 8, 8, 0, 0, None, None, None) == asd.ASD_E_INVALID_ARG
    assert f(ctypes.byref(q), 1, 1, 0, 8, 0, 0, None, None, None) == asd.ASD_E_INVALID_ARG
    assert f(ctypes.byref(bad), 1, 0, 8, 8, 0, 0, None, None, None) == asd.ASD_E_INVALID_ARG
    assert f(ctypes.byref(q), 1, 0, 8, 8, 0, 0, None, None, None) == asd.ASD_OK


def test_rectify_validation(lib):
    eye = (ctypes.c_double * 9)(1, 0, 0, 0, 1, 0, 0, 0, 1)
    sing = (ctypes.c_double * 9)(1, 2, 0, 2, 4, 0, 0, 0, 1)
    assert lib.asd_rectify(None, 0, 8, 8, None, None, None) == asd.ASD_E_INVALID_ARG
    assert lib.asd_rectify(sing, 0, 8, 8, None, None, None) == asd.ASD_E_INVALID_ARG
    assert lib.asd_rectify(eye, -1, 8, 8, None, None, None) == asd.ASD_E_INVALID_ARG
    assert lib.asd_rectify(eye, 0, 8, 8, None, None, None) == asd.ASD_OK


def test_binding_argument_checks():
    """The binding verifies dtype, shape, contiguity and placement before a raw
    pointer reaches the C ABI (no GPU needed: the checks run first)."""
    import torch
    st = asd.Stereo.__new__(asd.Stereo)
    st.params, st.device = asd.Params(64, 48, 16, census_w=5, census_h=5), 0
    u8 = torch.zeros(2, 48, 64, dtype=torch.uint8)
    f32 = torch.zeros(2, 48, 64)
    s32 = torch.zeros(2, 4, dtype=torch.int32)
    assert st._io(True, True, u8, u8, f32, f32, s32) == 2          # host path: CPU tensors ok
    with pytest.raises(ValueError):
        st._io(False, True, u8, u8, None, None)                     # device path: CPU tensor
    with pytest.raises(TypeError):
        st._io(True, True, u8.float(), u8, None, None)              # wrong dtype
    with pytest.raises(ValueError):
        st._io(True, True, u8, u8[:1], None, None)                  # right has fewer frames
    with pytest.raises(ValueError):
        st._io(True, True, u8, u8, f32[:, :, :32], None)            # wrong width
    with pytest.raises(ValueError):
        st._io(True, True, u8, u8.transpose(1, 2).contiguous().transpose(1, 2), None, None)
    with pytest.raises(ValueError):
        st._io(True, True, u8, u8, None, None, torch.zeros(3, 4, dtype=torch.int32))
    p = asd.Params(64, 48, 16, block_w=3, block_h=3)
    assert (p.p1, p.p2) == (72, 288)                                # S:388 scaled by the block area
    assert (asd.Params(64, 48, 16).p1, asd.Params(64, 48, 16).p2) == (8, 32)

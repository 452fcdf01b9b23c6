"""B200-native active-stereo depth engine (arXiv 2201.11924, SimSense stage).

The compute path is libasd.so (sm_100a CUDA kernels behind the C ABI in
include/asd.h); this package is its thin Python binding.  See DESIGN.md.
"""
from .abi import (ASD_E_CUDA, ASD_E_INVALID_ARG, ASD_E_OOM, ASD_E_UNSUPPORTED, ASD_OK,  # noqa: F401
                  MASK_BORDER, MASK_LR, MASK_NONPOS, MASK_UNIQUE, AsdError, Params, Stereo,
                  asd_frame_stats, load, rectify, register_depth, scratch_bytes, sensor_noise, SYMBOLS, LIB_PATH)

__all__ = ["Params", "Stereo", "AsdError", "load", "rectify", "register_depth", "scratch_bytes", "sensor_noise"]

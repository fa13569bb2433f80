"""ctypes binding of libpfb200.so (include/pf_b200.h) and status -> exception mapping.

The product path has no fallback: if the shared library is missing or a CUDA
device is absent, calls raise instead of computing anything on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import errors

# PF_B200_LIB: load another build of the same ABI (A/B timing of kernel variants)
_LIB_PATH = Path(os.environ.get("PF_B200_LIB") or Path(__file__).resolve().parent / "_lib" / "libpfb200.so")

PF_MAX_LEVELS = 12
PF_MAX_MPPS = 8
PF_MAX_CROPS = 16

PF_OK = 0
PF_ERR_INVALID_ARG = 1
PF_ERR_OUT_OF_BOUNDS = 2
PF_ERR_INTEGRITY = 3
PF_ERR_EXHAUSTED = 4
PF_ERR_NO_SAMPLABLE = 5
PF_ERR_CUDA = 6
PF_ERR_EMPTY_FOREGROUND = 7
PF_ERR_CAPACITY = 8
PF_ERR_INTERNAL = 9
PF_ERR_DECODE = 10

PF_U8, PF_F32, PF_BF16 = 0, 1, 2
PF_HWC, PF_NCHW = 0, 1
PF_SKIP_PASSTHROUGH = 256
PF_SKIP_RESAMPLED = 512
PF_MASK_LUMINANCE, PF_MASK_SATURATION = 0, 1

PF_AUG_FLIP, PF_AUG_JITTER, PF_AUG_GRAY, PF_AUG_BLUR, PF_AUG_SOLARIZE = 1, 2, 4, 8, 16


class SlideDesc(C.Structure):
    _fields_ = [
        ("level_ptr", C.c_uint64 * PF_MAX_LEVELS),
        ("tile_map", C.c_uint64 * PF_MAX_LEVELS),
        ("mpp", C.c_double * PF_MAX_LEVELS),
        ("width", C.c_int32 * PF_MAX_LEVELS),
        ("height", C.c_int32 * PF_MAX_LEVELS),
        ("tiles_x", C.c_int32 * PF_MAX_LEVELS),
        ("tiles_y", C.c_int32 * PF_MAX_LEVELS),
        ("downsample", C.c_int32 * PF_MAX_LEVELS),
        ("n_levels", C.c_int32),
        ("tile_size", C.c_int32),
        ("base_mpp", C.c_double),
        ("status_word", C.c_uint64),
    ]


class SamplerConfig(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64),
        ("key_slide", C.c_uint64),
        ("key_coords", C.c_uint64),
        ("key_mpp", C.c_uint64),
        ("min_foreground", C.c_double),
        ("mpp", C.c_double * PF_MAX_MPPS),
        ("mpp_weight", C.c_double * PF_MAX_MPPS),
        ("n_mpps", C.c_int32),
        ("patch_size", C.c_int32),
        ("max_attempts", C.c_int32),
        ("strategy", C.c_int32),
        ("n_slides", C.c_int32),
        ("grid", C.c_int32),
    ]


class SamplerSlide(C.Structure):
    _fields_ = [
        ("poly_blob", C.c_uint64),
        ("bbox", C.c_double * 4),
        ("weight", C.c_double),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("fp", C.c_int32 * PF_MAX_MPPS),
        ("x_lo", C.c_int32 * PF_MAX_MPPS),
        ("x_hi", C.c_int32 * PF_MAX_MPPS),
        ("y_lo", C.c_int32 * PF_MAX_MPPS),
        ("y_hi", C.c_int32 * PF_MAX_MPPS),
        ("level", C.c_int32 * PF_MAX_MPPS),
        ("side", C.c_int32 * PF_MAX_MPPS),
        ("_pad", C.c_int32),
        ("raster", C.c_uint64),
    ]


class SamplerState(C.Structure):
    _fields_ = [
        ("c_slide", C.c_uint64),
        ("c_coords", C.c_uint64),
        ("c_mpp", C.c_uint64),
        ("seq", C.c_int64),
        ("consecutive_failures", C.c_int64),
        ("attempts", C.c_int64),
        ("slow_evals", C.c_int64),
        ("status", C.c_int32),
        ("emitted", C.c_int32),
        ("cur_slide", C.c_int32),
        ("cur_used", C.c_int32),
        ("_reserved", C.c_int64),
    ]


class MultiCropConfig(C.Structure):
    _fields_ = [
        ("rrc_table_global", C.c_uint64),
        ("rrc_table_local", C.c_uint64),
        ("n_global", C.c_int32),
        ("n_local", C.c_int32),
        ("global_size", C.c_int32),
        ("local_size", C.c_int32),
        ("src_size", C.c_int32),
        ("blur_kernel", C.c_int32),
        ("global_scale", C.c_float * 2),
        ("local_scale", C.c_float * 2),
        ("ratio", C.c_float * 2),
        ("p_flip", C.c_float),
        ("p_jitter", C.c_float),
        ("p_gray", C.c_float),
        ("brightness", C.c_float),
        ("contrast", C.c_float),
        ("saturation", C.c_float),
        ("hue", C.c_float),
        ("sigma_min", C.c_float),
        ("sigma_max", C.c_float),
        ("solarize_threshold", C.c_float),
        ("p_blur", C.c_float * PF_MAX_CROPS),
        ("p_solarize", C.c_float * PF_MAX_CROPS),
    ]


# numpy mirrors of the device-array structs
SPEC_DTYPE = np.dtype(
    [
        ("seq", "<i8"), ("target_mpp", "<f8"), ("slide", "<i4"), ("x", "<i4"), ("y", "<i4"),
        ("width", "<i4"), ("height", "<i4"), ("out_size", "<i4"), ("mpp_idx", "<i4"),
        ("level", "<i4"), ("side", "<i4"), ("sx", "<i4"), ("sy", "<i4"), ("flags", "<i4"),
    ]
)
assert SPEC_DTYPE.itemsize == 64

CROP_DTYPE = np.dtype(
    [
        ("top", "<i4"), ("left", "<i4"), ("height", "<i4"), ("width", "<i4"), ("out_size", "<i4"),
        ("flags", "<i4"), ("order", "u1", (4,)), ("brightness", "<f4"), ("contrast", "<f4"),
        ("saturation", "<f4"), ("hue", "<f4"), ("sigma", "<f4"), ("solarize_threshold", "<f4"),
        ("patch", "<i4"), ("crop", "<i4"), ("_pad", "<i4"),
    ]
)
assert CROP_DTYPE.itemsize == 64

assert C.sizeof(SamplerState) == 80
assert C.sizeof(SlideDesc) == 96 + 96 + 96 + 5 * 48 + 8 + 8 + 8


class _Lib:
    _inst = None

    def __init__(self):
        if not _LIB_PATH.exists():
            raise errors.NativeLibraryError(
                f"{_LIB_PATH} is missing: run `python -m paper_2404_15217_b200.build` "
                "(there is no CPU fallback)"
            )
        self.lib = C.CDLL(str(_LIB_PATH))
        L = self.lib
        vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
        sig = {
            "pf_abi_version": ([], C.c_int),
            "pf_last_error": ([], C.c_char_p),
            "pf_launch_count": ([], u64),
            "pf_build_level": ([C.POINTER(SlideDesc), i32, i32, vp], C.c_int),
            "pf_thumbnail": ([C.POINTER(SlideDesc), i32, i32, vp, vp], C.c_int),
            "pf_plan_regions": ([vp, vp, i32, vp], C.c_int),
            "pf_read_regions": ([vp, vp, i32, i32, i32, i32, vp, vp, vp, vp], C.c_int),
            "pf_read_region_fits": ([i32, i32, i32, C.POINTER(i32)], C.c_int),
            "pf_host_alloc_mapped": ([i64, C.POINTER(vp), C.POINTER(vp)], C.c_int),
            "pf_host_free": ([vp], C.c_int),
            "pf_tier_prefetch": ([vp, vp, i32, vp, i32, i32, i32, i32, vp], C.c_int),
            "pf_slide_create": ([i32, i32, dbl, i32, i32, C.POINTER(vp)], C.c_int),
            "pf_slide_destroy": ([vp], C.c_int),
            "pf_slide_get_desc": ([vp, C.POINTER(SlideDesc)], C.c_int),
            "pf_slide_upload_level0": ([vp, vp, i64, i32, vp], C.c_int),
            "pf_slide_upload_tile": ([vp, i32, i32, i32, vp, i32, i32, vp], C.c_int),
            "pf_slide_build_pyramid": ([vp, vp], C.c_int),
            "pf_slide_status": ([C.POINTER(SlideDesc), i32, vp], C.c_int),
            "pf_read_region_generic_scratch_bytes": ([i32, i32, C.POINTER(i64)], C.c_int),
            "pf_read_region_generic": ([vp, vp, i32, i32, i32, vp, vp, vp, i64, vp, vp], C.c_int),
            "pf_normalize": ([vp, i64, i32, vp, vp, vp, vp], C.c_int),
            "pf_mask": ([vp, i32, i32, i32, dbl, i32, vp, vp, vp], C.c_int),
            "pf_polygon_trace": (
                [vp, i32, i32, dbl, dbl, vp, i64, vp, i32, C.POINTER(i64), C.POINTER(i32)],
                C.c_int,
            ),
            "pf_polygon_trace_device_scratch_bytes": ([i32, i32, C.POINTER(i64)], C.c_int),
            "pf_polygon_trace_device": (
                [vp, i32, i32, dbl, dbl, vp, i64, vp, i64, vp, i32, C.POINTER(i64), C.POINTER(i32), vp], C.c_int),
            "pf_polygon_index_size": ([vp, vp, i32, C.POINTER(i64)], C.c_int),
            "pf_polygon_index_build": ([vp, vp, i32, vp, i64], C.c_int),
            "pf_overlap_fraction": ([vp, vp, i32, i32, vp, vp], C.c_int),
            "pf_polygon_raster_bytes": ([vp, dbl, C.POINTER(i64)], C.c_int),
            "pf_polygon_raster_build": ([vp, vp, dbl, vp, i64, vp], C.c_int),
            "pf_sample_workspace_bytes": ([C.POINTER(SamplerConfig), i32, C.POINTER(i64)], C.c_int),
            "pf_sample": (
                [C.POINTER(SamplerConfig), vp, vp, vp, i32, vp, vp, i64, i32, i32, i32, vp],
                C.c_int,
            ),
            "pf_capped_draw": ([u64, vp, vp, i32, i32, vp, vp], C.c_int),
            "pf_png_inflate": ([vp, vp, i32, vp, vp, vp, vp, vp], C.c_int),
            "pf_jpeg_decode": ([vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, i32, vp, i64, i32, vp, vp], C.c_int),
            "pf_jpeg_struct_sizes": ([C.POINTER(i32), C.POINTER(i32)], C.c_int),
            "pf_jpeg_prepare": ([vp, vp, vp, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
            "pf_png_unfilter": ([vp, vp, vp, vp, vp, i32, i32, vp, vp], C.c_int),
            "pf_crop_params": ([u64, i32, u64, i32, C.POINTER(MultiCropConfig), vp, vp], C.c_int),
            "pf_multicrop": (
                [vp, vp, vp, i32, vp, C.POINTER(MultiCropConfig), i32, vp, vp, vp, vp, vp],
                C.c_int,
            ),
            "pf_philox4x32_10": ([vp, vp, vp], None),
            "pf_rrc_table_bytes": ([i32, i32, C.POINTER(i64)], C.c_int),
            "pf_rrc_table_build": ([i32, i32, vp, vp], C.c_int),
            "pf_synth_level0": ([C.POINTER(SlideDesc), vp, i32, i32, i32, C.c_float, u64, vp], C.c_int),
        }
        self.symbols = sorted(sig)
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        if L.pf_abi_version() != 3:
            raise errors.NativeLibraryError("libpfb200 ABI version mismatch")

    @classmethod
    def get(cls) -> "_Lib":
        if cls._inst is None:
            cls._inst = _Lib()
        return cls._inst


def lib():
    return _Lib.get().lib


def exported_symbols() -> list:
    return _Lib.get().symbols


def check(rc: int, what: str = "") -> None:
    if rc == PF_OK:
        return
    msg = lib().pf_last_error().decode("utf-8", "replace")
    if what:
        msg = f"{what}: {msg}"
    raise status_error(rc, msg)


def status_error(rc: int, msg: str) -> Exception:
    return {
        PF_ERR_INVALID_ARG: ValueError,
        PF_ERR_OUT_OF_BOUNDS: errors.OutOfBoundsError,
        PF_ERR_INTEGRITY: errors.IntegrityError,
        PF_ERR_EXHAUSTED: errors.ExhaustedAttemptsError,
        PF_ERR_NO_SAMPLABLE: errors.NoSamplableSlideError,
        PF_ERR_EMPTY_FOREGROUND: errors.EmptyForegroundError,
        PF_ERR_CAPACITY: errors.CapacityError,
        PF_ERR_DECODE: errors.DecodeError,
    }.get(rc, errors.NativeError)(msg)


def stream_ptr(stream=None) -> int:
    """Raw cudaStream_t of a torch stream (default: the current stream)."""
    import torch

    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise errors.NativeError("a CUDA device is required (the product path has no CPU fallback)")
    lib()  # load eagerly so a missing .so fails here
    return torch


def launches() -> int:
    return int(lib().pf_launch_count())


if os.environ.get("PF_B200_EAGER_LOAD"):
    lib()

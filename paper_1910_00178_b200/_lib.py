"""ctypes binding of the C-ABI in include/ngemm_cuda.h (libngemm_cuda.so, in-tree).

There is deliberately no fallback: if the shared library is missing this module raises
on first use, and every entry point reports CUDA errors as exceptions.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# NGEMM_LIB: an alternative in-tree build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("NGEMM_LIB") or os.path.join(_HERE, "lib", "libngemm_cuda.so")

# every symbol include/ngemm_cuda.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "ngemm_cuda_gemm_u8i8", "ngemm_cuda_gemm_u8i8_ex", "ngemm_cuda_repack", "ngemm_cuda_packed_validate",
    "ngemm_cuda_packed_upload", "ngemm_cuda_packed_from_device", "ngemm_cuda_packed_free",
    "ngemm_cuda_packed_info", "ngemm_cuda_gemm_packed", "ngemm_cuda_gemm_u8i8_host",
    "ngemm_cuda_gemm_packed_host", "ngemm_cuda_shard_rows", "ngemm_cuda_gemm_u8i8_multi", "ngemm_cuda_free",
    "ngemm_cuda_abi_version", "ngemm_cuda_status_name", "ngemm_cuda_last_error", "ngemm_cuda_pick_kernel",
    "ngemm_cuda_launch_count", "ngemm_cuda_gemm_i16", "ngemm_cuda_gemm_i16_host", "ngemm_cuda_gemm_packed_i16",
    "ngemm_cuda_gemm_packed_resident_host", "ngemm_cuda_device", "ngemm_cuda_tune", "ngemm_cuda_tune_store_save",
    "ngemm_cuda_tune_store_load", "ngemm_cuda_tune_clear", "ngemm_cuda_gemm_u8i8_strided_batched",
    "ngemm_cuda_gemm_u8i8_requant", "ngemm_cuda_set_option", "ngemm_cuda_get_option", "ngemm_cuda_reset_options",
    "ngemm_cuda_trim", "ngemm_cuda_packed_upload_sharded", "ngemm_cuda_gemm_packed_multi",
]

OK, ERR_SHAPE, ERR_UNSUPPORTED, ERR_CONFIG, ERR_RANGE, ERR_CORRUPTION, ERR_INDEX, ERR_CUDA, ERR_TUNE = range(9)
KERNEL_AUTO, KERNEL_TCGEN05, KERNEL_SIMT, KERNEL_SKINNY, KERNEL_SAT_HYBRID = range(5)
KERNEL_NAMES = {KERNEL_AUTO: "auto", KERNEL_TCGEN05: "tcgen05", KERNEL_SIMT: "simt", KERNEL_SKINNY: "skinny",
                KERNEL_SAT_HYBRID: "sat_hybrid"}


class PackedMeta(C.Structure):
    _fields_ = [("w", C.c_int32), ("h", C.c_int32), ("v", C.c_int32),
                ("tm", C.c_int64), ("tn", C.c_int64), ("tk", C.c_int64),
                ("perm", C.c_int32), ("m_orig", C.c_int64), ("k_orig", C.c_int64),
                ("m_pad", C.c_int64), ("k_pad", C.c_int64)]


class TuneRecord(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64), ("sat_mode", C.c_int32),
                ("kernel", C.c_int32), ("tc_cfg", C.c_int32), ("tc_splits", C.c_int32),
                ("skinny_variant", C.c_int32), ("median_ns", C.c_double), ("min_ns", C.c_double),
                ("trials", C.c_int32), ("timestamp", C.c_int64)]


_lock = threading.Lock()
_lib = None


def load():
    """Load libngemm_cuda.so (raises if it was not built — no CPU fallback exists)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libngemm_cuda.so not built ({LIB_PATH}); run `make` or __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        i64, vp, i32 = C.c_int64, C.c_void_p, C.c_int
        st = C.c_int
        L.ngemm_cuda_gemm_u8i8.argtypes = [vp, i64, vp, i64, vp, i64, i64, i64, i64, i32, vp]
        L.ngemm_cuda_gemm_u8i8_ex.argtypes = [vp, i64, vp, i64, vp, i64, i64, i64, i64, i32, i32, vp]
        L.ngemm_cuda_gemm_u8i8_strided_batched.argtypes = [vp, i64, i64, vp, i64, i64, vp, i64, i64, i64, i64, i64,
                                                            i64, i32, vp]
        L.ngemm_cuda_gemm_u8i8_requant.argtypes = [vp, i64, vp, i64, vp, i64, i64, i64, i64, vp, vp, i32, i32, vp]
        L.ngemm_cuda_repack.argtypes = [C.POINTER(PackedMeta), vp, vp, i64, vp]
        L.ngemm_cuda_packed_validate.argtypes = [C.POINTER(PackedMeta)]
        L.ngemm_cuda_packed_upload.argtypes = [C.POINTER(PackedMeta), vp, C.c_size_t, C.POINTER(vp)]
        L.ngemm_cuda_packed_from_device.argtypes = [vp, i64, i64, i64, C.POINTER(vp)]
        L.ngemm_cuda_packed_free.argtypes = [vp]
        L.ngemm_cuda_packed_info.argtypes = [vp, C.POINTER(vp), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64),
                                             C.POINTER(i32)]
        L.ngemm_cuda_gemm_packed.argtypes = [vp, vp, i64, vp, i64, i64, i32, vp]
        L.ngemm_cuda_gemm_u8i8_host.argtypes = [vp, vp, vp, i64, i64, i64, i32, i32]
        L.ngemm_cuda_gemm_packed_host.argtypes = [C.POINTER(PackedMeta), vp, C.c_size_t, vp, vp, i64, i32, i32]
        L.ngemm_cuda_shard_rows.argtypes = [i64, i32, i64, C.POINTER(i64)]
        L.ngemm_cuda_gemm_u8i8_multi.argtypes = [C.POINTER(i32), i32, vp, vp, vp, i64, i64, i64, i32, i32,
                                                 C.POINTER(vp)]
        L.ngemm_cuda_free.argtypes = [vp]
        L.ngemm_cuda_gemm_i16.argtypes = [vp, i64, vp, i64, vp, i64, i64, i64, i64, vp]
        L.ngemm_cuda_gemm_i16_host.argtypes = [vp, vp, vp, i64, i64, i64]
        L.ngemm_cuda_gemm_packed_i16.argtypes = [vp, vp, i64, vp, i64, i64, vp]
        L.ngemm_cuda_gemm_packed_resident_host.argtypes = [vp, vp, vp, i64, i32]
        L.ngemm_cuda_device.argtypes = [C.POINTER(i32)]
        L.ngemm_cuda_tune.argtypes = [i64, i64, i64, i32, i32, i32, C.POINTER(TuneRecord)]
        L.ngemm_cuda_tune_store_save.argtypes = [C.c_char_p]
        L.ngemm_cuda_tune_store_load.argtypes = [C.c_char_p, C.POINTER(i32)]
        L.ngemm_cuda_tune_clear.argtypes = []
        if hasattr(L, "ngemm_cuda_set_option"):  # absent only in older builds loaded for A/B runs
            L.ngemm_cuda_set_option.argtypes = [C.c_char_p, i32]
            L.ngemm_cuda_get_option.argtypes = [C.c_char_p]
            L.ngemm_cuda_reset_options.argtypes = []
            L.ngemm_cuda_trim.argtypes = []
            L.ngemm_cuda_packed_upload_sharded.argtypes = [C.POINTER(PackedMeta), vp, C.c_size_t, C.POINTER(i32), i32,
                                                           C.POINTER(vp)]
            L.ngemm_cuda_gemm_packed_multi.argtypes = [C.POINTER(vp), i32, vp, vp, i64, i32]
        for f in EXPORTS:
            if os.environ.get("NGEMM_LIB") and not hasattr(L, f):
                continue  # A/B against an older build (experiments only)
            fn = getattr(L, f)
            if f not in ("ngemm_cuda_abi_version", "ngemm_cuda_status_name", "ngemm_cuda_last_error",
                         "ngemm_cuda_pick_kernel", "ngemm_cuda_launch_count", "ngemm_cuda_get_option"):
                fn.restype = st
        L.ngemm_cuda_abi_version.restype = C.c_int
        L.ngemm_cuda_status_name.argtypes = [C.c_int]
        L.ngemm_cuda_status_name.restype = C.c_char_p
        L.ngemm_cuda_last_error.restype = C.c_char_p
        L.ngemm_cuda_pick_kernel.argtypes = [i64, i64, i64, i32]
        L.ngemm_cuda_pick_kernel.restype = C.c_int
        L.ngemm_cuda_launch_count.restype = C.c_uint64
        if hasattr(L, "ngemm_cuda_get_option"):
            L.ngemm_cuda_get_option.restype = C.c_int
        _lib = L
        return L


class NgemmError(RuntimeError):
    """Base of the typed errors (the reference's ngemm::Error, common.hpp:77-79)."""


class ShapeError(NgemmError):
    pass


class UnsupportedError(NgemmError):
    pass


class ConfigError(NgemmError):
    pass


class RangeError(NgemmError):
    pass


class CorruptionError(NgemmError):
    pass


class IndexError_(NgemmError):
    pass


class CudaError(NgemmError):
    pass


class TuneError(NgemmError):
    pass


_ERRORS = {ERR_SHAPE: ShapeError, ERR_UNSUPPORTED: UnsupportedError, ERR_CONFIG: ConfigError,
           ERR_RANGE: RangeError, ERR_CORRUPTION: CorruptionError, ERR_INDEX: IndexError_, ERR_CUDA: CudaError,
           ERR_TUNE: TuneError}


def check(status: int):
    if status != OK:
        L = load()
        msg = L.ngemm_cuda_last_error().decode(errors="replace")
        raise _ERRORS.get(status, NgemmError)(msg or L.ngemm_cuda_status_name(status).decode())


def launch_count() -> int:
    return int(load().ngemm_cuda_launch_count())


def set_option(name: str, value: int):
    """Experiment / test knob (include/ngemm_cuda.h): e.g. set_option("TC_CFG", 2)."""
    check(load().ngemm_cuda_set_option(name.encode(), int(value)))


def get_option(name: str) -> int:
    return int(load().ngemm_cuda_get_option(name.encode()))


def reset_options():
    check(load().ngemm_cuda_reset_options())


class options:
    """Context manager: `with _lib.options(TC_CFG=2, TC_SPLITS=1): ...` restores the knobs after."""

    def __init__(self, **kv):
        self.kv = kv
        self.saved = {}

    def __enter__(self):
        for k, v in self.kv.items():
            self.saved[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.saved.items():
            set_option(k, v)

"""ctypes front end for the CPU oracle (TEST INFRASTRUCTURE ONLY).

`Oracle` wraps oracle/liboracle.so (our C restatement of the reference path, see
oracle.h for the file:line each function follows).  `Reference` wraps oracle/_ref/
libngemm_ref.so, the unmodified reference compiled from its own headers (ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference legs
import this module, and only as the checker or the reported CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libngemm_ref.so")

SAT, EXACT = 0, 1  # reference SatMode order (lanes.hpp:18)


def _p(a):
    return C.c_void_p(a.ctypes.data)


class PackedMeta(C.Structure):
    _fields_ = [("w", C.c_int32), ("h", C.c_int32), ("v", C.c_int32),
                ("tm", C.c_int64), ("tn", C.c_int64), ("tk", C.c_int64),
                ("perm", C.c_int32), ("m_orig", C.c_int64), ("k_orig", C.c_int64),
                ("m_pad", C.c_int64), ("k_pad", C.c_int64)]


class Oracle:
    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            subprocess.check_call(["make", "-s", "-C", _HERE, os.path.abspath(path)])
        L = C.CDLL(path)
        i64, u64, vp = C.c_int64, C.c_uint64, C.c_void_p
        L.ngo_mat_random_u8.argtypes = [vp, i64, i64, u64, i64, i64]
        L.ngo_mat_random_i8.argtypes = [vp, i64, i64, u64, i64, i64]
        L.ngo_mat_normal_i8.argtypes = [vp, i64, i64, u64, C.c_double]
        L.ngo_mat_random_i16.argtypes = [vp, i64, i64, u64, i64, i64]
        L.ngo_gemm.argtypes = [vp, i64, vp, i64, vp, i64, i64, i64, i64, C.c_int, C.c_int]
        L.ngo_gemm_i16.argtypes = [vp, i64, vp, i64, vp, i64, i64, i64, i64]
        L.ngo_madd_pair.argtypes = [C.c_uint8, C.c_uint8, C.c_int8, C.c_int8, C.c_int]
        L.ngo_madd_pair.restype = C.c_int32
        L.ngo_packed_init.argtypes = [C.POINTER(PackedMeta), C.c_int32, C.c_int32, C.c_int32,
                                      i64, i64, i64, C.c_int32, i64, i64]
        L.ngo_packed_init.restype = C.c_int
        L.ngo_packed_elem_offset.argtypes = [C.POINTER(PackedMeta), i64, i64]
        L.ngo_packed_elem_offset.restype = i64
        L.ngo_pack_u8.argtypes = [C.POINTER(PackedMeta), vp, i64, vp]
        L.ngo_unpack_u8.argtypes = [C.POINTER(PackedMeta), vp, vp, i64]
        L.ngo_unpack_u8.restype = i64
        L.ngo_fnv1a.argtypes = [vp, C.c_size_t]
        L.ngo_fnv1a.restype = u64
        L.ngo_rng_next_in.argtypes = [vp, i64, i64]
        L.ngo_rng_next_in.restype = i64
        self.L = L

    # -- inputs --------------------------------------------------------------------------
    def mat_random_u8(self, rows, cols, seed, lo=0, hi=255):
        out = np.empty((rows, cols), np.uint8)
        self.L.ngo_mat_random_u8(_p(out), rows, cols, seed, lo, hi)
        return out

    def mat_random_i8(self, rows, cols, seed, lo=-128, hi=127):
        out = np.empty((rows, cols), np.int8)
        self.L.ngo_mat_random_i8(_p(out), rows, cols, seed, lo, hi)
        return out

    def mat_random_i16(self, rows, cols, seed, lo=-32768, hi=32767):
        out = np.empty((rows, cols), np.int16)
        self.L.ngo_mat_random_i16(_p(out), rows, cols, seed, lo, hi)
        return out

    def mat_normal_i8(self, rows, cols, seed, sigma=32.0):
        out = np.empty((rows, cols), np.int8)
        self.L.ngo_mat_normal_i8(_p(out), rows, cols, seed, sigma)
        return out

    # -- oracles -------------------------------------------------------------------------
    def gemm(self, a: np.ndarray, b: np.ndarray, mode: int, threads: int | None = None):
        """C[m][n] per gemm_ref (mode 1) or gemm_sat_oracle (mode 0)."""
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.int8)
        m, k = a.shape
        n, kb = b.shape
        assert k == kb
        c = np.empty((m, n), np.int32)
        if threads is None:
            threads = max(1, min(os.cpu_count() or 1, 64))
        self.L.ngo_gemm(_p(a), k, _p(b), k, _p(c), n, m, n, k, mode, threads)
        return c

    def gemm_i16(self, a: np.ndarray, b: np.ndarray):
        """C[m][n] per gemm_ref on i16 x i16 (sum of products mod 2^32)."""
        a = np.ascontiguousarray(a, np.int16)
        b = np.ascontiguousarray(b, np.int16)
        m, k = a.shape
        n, kb = b.shape
        assert k == kb
        c = np.empty((m, n), np.int32)
        self.L.ngo_gemm_i16(_p(a), k, _p(b), k, _p(c), n, m, n, k)
        return c

    def madd_pair(self, a0, a1, b0, b1, mode):
        return self.L.ngo_madd_pair(a0, a1, b0, b1, mode)

    # -- layout --------------------------------------------------------------------------
    def packed_meta(self, m, k, w=64, h=4, v=16, tm=None, tn=64, tk=None, perm=0):
        meta = PackedMeta()
        tm = v if tm is None else tm
        tk = h if tk is None else tk
        rc = self.L.ngo_packed_init(C.byref(meta), w, h, v, tm, tn, tk, perm, m, k)
        if rc != 0:
            raise ValueError(f"invalid packed config rc={rc}")
        return meta

    def pack(self, a: np.ndarray, meta: PackedMeta) -> np.ndarray:
        a = np.ascontiguousarray(a, np.uint8)
        out = np.empty(meta.m_pad * meta.k_pad, np.uint8)
        self.L.ngo_pack_u8(C.byref(meta), _p(a), a.shape[1], _p(out))
        return out

    def unpack(self, packed: np.ndarray, meta: PackedMeta) -> np.ndarray:
        a = np.zeros((meta.m_orig, meta.k_orig), np.uint8)
        packed = np.ascontiguousarray(packed)
        rc = self.L.ngo_unpack_u8(C.byref(meta), _p(packed), _p(a), meta.k_orig)
        if rc != 0:
            raise ValueError(f"nonzero padding at flat index {rc - 1}")
        return a

    def elem_offset(self, meta, gm, gk):
        return self.L.ngo_packed_elem_offset(C.byref(meta), gm, gk)

    def fnv1a(self, arr: np.ndarray) -> int:
        arr = np.ascontiguousarray(arr)
        return int(self.L.ngo_fnv1a(_p(arr), arr.nbytes))


class Reference:
    """The unmodified reference (oracle/_ref), reachable only where it was built."""

    VARIANTS = {"gemm_ref": 0, "gemm_sat_oracle": 1, "gemm_conventional": 2, "gemm_ngemm": 3}

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        i64, vp = C.c_int64, C.c_void_p
        L.ref_host_isa_bits.restype = C.c_int
        L.ref_mat_random.argtypes = [C.c_int, i64, i64, C.c_uint64, i64, i64, vp]
        L.ref_gemm.argtypes = [C.c_int, vp, vp, vp, i64, i64, i64, C.c_int, C.c_int, C.c_int]
        L.ref_gemm_i16.argtypes = [C.c_int, vp, vp, vp, i64, i64, i64]
        L.ref_gemm.restype = C.c_int
        L.ref_pack.argtypes = [vp, i64, i64, C.c_int, C.c_int, C.c_int, i64, i64, i64, C.c_int, vp, i64]
        L.ref_pack.restype = i64
        L.ref_gemm_ngemm_packed.argtypes = [vp, i64, C.c_int, C.c_int, C.c_int, i64, i64, i64, C.c_int,
                                            i64, i64, vp, i64, vp, C.c_int, C.c_int]
        L.ref_gemm_ngemm_packed.restype = C.c_int
        L.ref_session_create.argtypes = [vp, vp, i64, i64, i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_session_create.restype = vp
        L.ref_session_run.argtypes = [vp]
        L.ref_session_run.restype = C.c_int
        L.ref_session_result.argtypes = [vp, vp]
        L.ref_session_destroy.argtypes = [vp]
        self.L = L

    @staticmethod
    def available(path: str = REF_PATH) -> bool:
        return os.path.exists(path)

    def host_isa_bits(self) -> int:
        return self.L.ref_host_isa_bits()

    def mat_random(self, kind: int, rows, cols, seed, lo, hi):
        out = np.empty((rows, cols), {0: np.uint8, 1: np.int8, 2: np.int16, 3: np.int32}[kind])
        self.L.ref_mat_random(kind, rows, cols, seed, lo, hi, _p(out))
        return out

    def gemm(self, variant: str, a, b, mode=EXACT, engine=0, isa_bits=None):
        a = np.ascontiguousarray(a, np.uint8)
        b = np.ascontiguousarray(b, np.int8)
        m, k = a.shape
        n = b.shape[0]
        c = np.empty((m, n), np.int32)
        isa_bits = self.host_isa_bits() if isa_bits is None else isa_bits
        rc = self.L.ref_gemm(self.VARIANTS[variant], _p(a), _p(b), _p(c), m, n, k, mode, engine, isa_bits)
        if rc != 0:
            raise RuntimeError(f"reference {variant} failed rc={rc}")
        return c

    def gemm_i16(self, variant: str, a, b):
        a = np.ascontiguousarray(a, np.int16)
        b = np.ascontiguousarray(b, np.int16)
        m, k = a.shape
        n = b.shape[0]
        c = np.empty((m, n), np.int32)
        rc = self.L.ref_gemm_i16({"gemm_ref": 0, "gemm_conventional": 2}[variant], _p(a), _p(b), _p(c), m, n, k)
        if rc != 0:
            raise RuntimeError(f"reference i16 {variant} failed rc={rc}")
        return c

    def pack(self, a, w, h, v, tm, tn, tk, perm):
        a = np.ascontiguousarray(a, np.uint8)
        m, k = a.shape
        cap = (m + tm) * (k + tk)
        out = np.empty(cap, np.uint8)
        nb = self.L.ref_pack(_p(a), m, k, w, h, v, tm, tn, tk, perm, _p(out), cap)
        if nb < 0:
            raise ValueError("reference pack_weights rejected the config")
        return out[:nb].copy()

    def gemm_ngemm_packed(self, packed, meta, b, mode, engine=1):
        b = np.ascontiguousarray(b, np.int8)
        n = b.shape[0]
        c = np.empty((meta.m_orig, n), np.int32)
        rc = self.L.ref_gemm_ngemm_packed(_p(packed), packed.nbytes, meta.w, meta.h, meta.v, meta.tm, meta.tn,
                                          meta.tk, meta.perm, meta.m_orig, meta.k_orig, _p(b), n, _p(c), mode,
                                          engine)
        if rc != 0:
            raise RuntimeError(f"reference gemm_ngemm failed rc={rc}")
        return c

    def session(self, a, b, variant: str, mode=EXACT, engine=0, isa_bits=None, threads=1):
        return RefSession(self, a, b, variant, mode, engine, isa_bits, threads)


class RefSession:
    """Prebuilt, row-sharded reference call for timing (the harness is ours)."""

    def __init__(self, ref: Reference, a, b, variant, mode, engine, isa_bits, threads):
        self.ref = ref
        self.a = np.ascontiguousarray(a, np.uint8)
        self.b = np.ascontiguousarray(b, np.int8)
        self.m, k = self.a.shape
        self.n = self.b.shape[0]
        isa_bits = ref.host_isa_bits() if isa_bits is None else isa_bits
        self.h = ref.L.ref_session_create(_p(self.a), _p(self.b), self.m, self.n, k,
                                          Reference.VARIANTS[variant], mode, engine, isa_bits, threads)

    def run(self):
        rc = self.ref.L.ref_session_run(self.h)
        if rc != 0:
            raise RuntimeError(f"reference session failed rc={rc}")

    def result(self):
        c = np.empty((self.m, self.n), np.int32)
        self.ref.L.ref_session_result(self.h, _p(c))
        return c

    def close(self):
        if self.h:
            self.ref.L.ref_session_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

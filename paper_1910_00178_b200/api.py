"""Python mirror of the reference's public GEMM API (proj/include/ngemm), backed by the C-ABI.

Names, argument meaning and error behaviour follow the reference so the parity tests read
like the reference's own tests (test_gemm.cpp, test_layout.cpp):

  reference (C++)                                        here
  SatMode {HardwareSaturating, WideningExact}            SatMode.HARDWARE_SATURATING / WIDENING_EXACT
  Engine {Auto, Emulated, Native}   (isa.hpp:59)         Engine.AUTO / EMULATED / NATIVE / CUDA
  KernelShape, kernel_shape (layout.hpp:21-39)           KernelShape, kernel_shape
  TileConfig, Perm (layout.hpp:54-108)                   TileConfig, Perm
  PackedWeight (layout.hpp:120-182)                      PackedWeight
  pack_weights / unpack_weights (layout.hpp:252-276)     pack_weights / unpack_weights
  gemm_conventional (gemm.hpp:327-369)                   gemm_conventional
  gemm_ngemm (gemm.hpp:373-409)                          gemm_ngemm

Engine mapping (no CPU fallback): AUTO and CUDA run the GPU dispatcher;
EMULATED runs the lane-faithful CUDA-core kernel; NATIVE raises UnsupportedError (the
product has no x86 SIMD path).  pack/unpack are the reference's offline host-side layout
steps and stay on the host; every multiply-accumulate runs in libngemm_cuda.so.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import (ConfigError, CorruptionError, CudaError, IndexError_, NgemmError, RangeError, ShapeError,
                   TuneError, UnsupportedError, check)


class SatMode(enum.IntEnum):
    HARDWARE_SATURATING = 0
    WIDENING_EXACT = 1


class Engine(enum.IntEnum):
    AUTO = 0
    EMULATED = 1
    NATIVE = 2
    CUDA = 3


class Perm(enum.IntEnum):
    MNK = 0
    MKN = 1
    NMK = 2
    NKM = 3
    KMN = 4
    KNM = 5


def m_before_k(p: Perm) -> bool:  # layout.hpp:77-79
    return p in (Perm.MNK, Perm.MKN, Perm.NMK)


@dataclass(frozen=True)
class KernelShape:
    w: int
    h: int
    v: int


def kernel_shape(vector_bits: int, elem_bits: int = 8) -> KernelShape:
    """layout.hpp:29-39 (isa given by its vector width: 128 scalar, 256 V256, 512 V512)."""
    if elem_bits not in (8, 16):
        raise UnsupportedError(f"kernel_shape: no kernel path for {elem_bits}-bit elements")
    w = vector_bits // elem_bits
    h = 4 if elem_bits == 8 else 2
    return KernelShape(w, h, w // h)


@dataclass(frozen=True)
class TileConfig:
    tm: int
    tn: int
    tk: int
    permutation: Perm = Perm.MNK

    def validate(self, shape: KernelShape):  # layout.hpp:92-102
        if self.tm < shape.v or self.tm % shape.v != 0:
            raise ConfigError(f"tile: tm={self.tm} is not a positive multiple of v={shape.v}")
        if self.tk < shape.h or self.tk % shape.h != 0:
            raise ConfigError(f"tile: tk={self.tk} is not a positive multiple of h={shape.h}")
        if self.tn < 1:
            raise ConfigError("tile: tn must be >= 1")


def _round_up(x, m):
    return (x + m - 1) // m * m


class PackedWeight:
    """Marshalled weight matrix (layout.hpp:110-182): padded m_pad x k_pad bytes in the
    two-level (tiled outer, v x h inner) order.  `upload()` makes the device-resident copy."""

    def __init__(self, shape: KernelShape, tile: TileConfig, m_orig: int, k_orig: int, data: np.ndarray | None = None):
        self.shape, self.tile = shape, tile
        self.m_orig, self.k_orig = int(m_orig), int(k_orig)
        self.m_pad, self.k_pad = _round_up(self.m_orig, tile.tm), _round_up(self.k_orig, tile.tk)
        self.data = np.zeros(self.m_pad * self.k_pad, np.uint8) if data is None else data
        self._dev = None

    def meta(self) -> _lib.PackedMeta:
        return _lib.PackedMeta(self.shape.w, self.shape.h, self.shape.v, self.tile.tm, self.tile.tn, self.tile.tk,
                               int(self.tile.permutation), self.m_orig, self.k_orig, self.m_pad, self.k_pad)

    def block_offset(self, m_blk, k_blk):  # layout.hpp:152-165 (vectorised)
        s, t = self.shape, self.tile
        tile_m = m_blk * s.v // t.tm
        tile_k = k_blk * s.h // t.tk
        bm = m_blk - tile_m * (t.tm // s.v)
        bk = k_blk - tile_k * (t.tk // s.h)
        tiles_m, tiles_k = self.m_pad // t.tm, self.k_pad // t.tk
        tile_lin = tile_m * tiles_k + tile_k if m_before_k(t.permutation) else tile_k * tiles_m + tile_m
        blocks_per_tile = (t.tm // s.v) * (t.tk // s.h)
        return (tile_lin * blocks_per_tile + bm * (t.tk // s.h) + bk) * s.w

    def elem_offset(self, gm, gk):  # layout.hpp:167-171
        s = self.shape
        return self.block_offset(gm // s.v, gk // s.h) + (gm % s.v) * s.h + gk % s.h

    def invalidate(self):
        """Call after mutating `data` in place: drops the cached device copy."""
        if self._dev is not None:
            self._dev.free()
            self._dev = None

    def upload(self) -> "DevicePackedWeight":
        if self._dev is None:
            self._dev = DevicePackedWeight.from_packed(self)
        return self._dev


def _rows_chunks(m, k):
    step = max(1, (1 << 24) // max(k, 1))
    for r0 in range(0, m, step):
        yield r0, min(m, r0 + step)


def pack_weights(a: np.ndarray, shape: KernelShape, tile: TileConfig) -> PackedWeight:
    """layout.hpp:252-270 (u8 path).  Offline host-side layout step."""
    a = np.asarray(a)
    if a.dtype != np.uint8:
        raise UnsupportedError(f"pack_weights: no kernel path for {a.dtype}")
    if shape.v * shape.h != shape.w or shape.h != 4:
        raise ConfigError(f"pack_weights: shape (w={shape.w},h={shape.h},v={shape.v}) does not match the u8 path")
    tile.validate(shape)
    m, k = a.shape
    p = PackedWeight(shape, tile, m, k)
    gk = np.arange(k, dtype=np.int64)
    for r0, r1 in _rows_chunks(m, k):
        gm = np.arange(r0, r1, dtype=np.int64)[:, None]
        p.data[p.elem_offset(gm, gk[None, :])] = a[r0:r1]
    return p


def unpack_weights(p: PackedWeight) -> np.ndarray:
    """layout.hpp:272-276 with the padding check of layout.hpp:231-248."""
    a = np.empty((p.m_orig, p.k_orig), np.uint8)
    gk = np.arange(p.k_pad, dtype=np.int64)
    for r0, r1 in _rows_chunks(p.m_pad, p.k_pad):
        gm = np.arange(r0, r1, dtype=np.int64)[:, None]
        vals = p.data[p.elem_offset(gm, gk[None, :])]
        pad = np.ones_like(vals, dtype=bool)
        rr = min(r1, p.m_orig) - r0
        if rr > 0:
            pad[:rr, :p.k_orig] = False
            a[r0:r0 + rr] = vals[:rr, :p.k_orig]
        bad = np.argwhere(pad & (vals != 0))
        if bad.size:
            r, c = bad[0]
            raise CorruptionError(f"nonzero value at padded coordinate ({r0 + r}, {c})")
    return a


def _engine_kernel(engine: Engine) -> int:
    engine = Engine(engine)
    if engine == Engine.NATIVE:
        raise UnsupportedError("no native path for this shape/mode on this host (the B200 engine is Engine::Cuda)")
    return _lib.KERNEL_SIMT if engine == Engine.EMULATED else _lib.KERNEL_AUTO


def _check_operands(a: np.ndarray, b: np.ndarray):  # gemm.hpp:19-30
    u8i8 = a.dtype == np.uint8 and b.dtype == np.int8
    i16 = a.dtype == np.int16 and b.dtype == np.int16
    if not (u8i8 or i16):
        raise UnsupportedError(f"gemm: no kernel path for {a.dtype} x {b.dtype}")
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[1]:
        raise ShapeError(f"gemm: K mismatch, A is {a.shape} but B is {b.shape} (B is stored [N x K])")


def gemm_conventional(a: np.ndarray, b: np.ndarray, shape: KernelShape, mode: SatMode,
                      engine: Engine = Engine.AUTO) -> np.ndarray:
    """gemm.hpp:327-369: C[m][n] = sum_k a[m][k] * b[n][k] on the GPU; host arrays in/out."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    _check_operands(a, b)
    if shape.v * shape.h != shape.w or shape.h != (4 if a.dtype == np.uint8 else 2):
        raise ShapeError("gemm_conventional: kernel shape does not match operand kind")
    kernel = _engine_kernel(engine)
    m, k = a.shape
    n = b.shape[0]
    c = np.empty((m, n), np.int32)
    if a.dtype == np.int16:  # the 16-bit path has no saturation stage (gemm.hpp:161-190)
        check(_lib.load().ngemm_cuda_gemm_i16_host(a.ctypes.data, b.ctypes.data, c.ctypes.data, m, n, k))
        return c
    check(_lib.load().ngemm_cuda_gemm_u8i8_host(a.ctypes.data, b.ctypes.data, c.ctypes.data, m, n, k, int(mode),
                                                  kernel))
    return c


def gemm_ngemm(p: PackedWeight, b: np.ndarray, mode: SatMode, engine: Engine = Engine.AUTO) -> np.ndarray:
    """gemm.hpp:373-409 on a prepacked weight; host arrays in/out (packed bytes repacked on device)."""
    b = np.ascontiguousarray(b)
    if b.dtype != np.int8:
        raise UnsupportedError(f"gemm_ngemm: no kernel path for u8 x {b.dtype}")
    if b.ndim != 2 or b.shape[1] != p.k_orig:
        raise ShapeError(f"gemm_ngemm: packed K={p.k_orig} but B has K={b.shape[-1]}")
    kernel = _engine_kernel(engine)
    n = b.shape[0]
    c = np.empty((p.m_orig, n), np.int32)
    data = np.ascontiguousarray(p.data)
    meta = p.meta()
    check(_lib.load().ngemm_cuda_gemm_packed_host(C.byref(meta), data.ctypes.data, data.nbytes, b.ctypes.data,
                                                    c.ctypes.data, n, int(mode), kernel))
    return c


# ------------------------------------------------------------------ device-resident API
def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return int(getattr(stream, "cuda_stream", stream))


def gemm_device(a, b, c=None, mode: SatMode = SatMode.WIDENING_EXACT, kernel: int = _lib.KERNEL_AUTO, stream=None):
    """C = A * B^T on CUDA torch tensors (A uint8 [M,K], B int8 [N,K], C int32 [M,N]); async on `stream`."""
    import torch
    if a.dtype != torch.uint8 or b.dtype != torch.int8:
        raise UnsupportedError(f"gemm: no kernel path for {a.dtype} x {b.dtype}")
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[1]:
        raise ShapeError(f"gemm: K mismatch, A is {tuple(a.shape)} but B is {tuple(b.shape)}")
    if a.stride(1) != 1 or b.stride(1) != 1:
        raise ShapeError("gemm: operands must be K-contiguous")
    m, k = a.shape
    n = b.shape[0]
    if c is None:
        c = torch.empty((m, n), dtype=torch.int32, device=a.device)
    if c.dtype != torch.int32 or tuple(c.shape) != (m, n) or c.stride(1) != 1:
        raise ShapeError("gemm: C must be int32 [M, N] with unit column stride")
    check(_lib.load().ngemm_cuda_gemm_u8i8_ex(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), c.data_ptr(),
                                                c.stride(0), m, n, k, int(mode), int(kernel), _stream_ptr(stream)))
    return c


def gemm_device_requant(a, b, scale, bias=None, zero_point: int = 0, out=None,
                        mode: SatMode = SatMode.WIDENING_EXACT, stream=None):
    """int8 out[M, N] = clamp(rint(float(A.B^T + bias) * scale) + zero_point) on CUDA tensors, the
    requantisation fused into the tcgen05 epilogue for exact mode and M > 16
    (ngemm_cuda_gemm_u8i8_requant).  scale: float32 [N], bias: int32 [N] or None."""
    import torch
    if a.dtype != torch.uint8 or b.dtype != torch.int8:
        raise UnsupportedError(f"gemm: no kernel path for {a.dtype} x {b.dtype}")
    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[1]:
        raise ShapeError(f"gemm: K mismatch, A is {tuple(a.shape)} but B is {tuple(b.shape)}")
    if a.stride(1) != 1 or b.stride(1) != 1:
        raise ShapeError("gemm: operands must be K-contiguous")
    m, k = a.shape
    n = b.shape[0]
    if scale.dtype != torch.float32 or tuple(scale.shape) != (n,) or (bias is not None and
                                                                    (bias.dtype != torch.int32 or
                                                                     tuple(bias.shape) != (n,))):
        raise ShapeError("requant: scale must be float32 [N] and bias int32 [N]")
    if not scale.is_contiguous() or (bias is not None and not bias.is_contiguous()):
        raise ShapeError("requant: scale and bias must be contiguous")
    for t in (b, scale) + ((bias,) if bias is not None else ()):
        if t.device != a.device:
            raise ShapeError(f"requant: operands must live on {a.device}, got one on {t.device}")
    if out is None:
        out = torch.empty((m, n), dtype=torch.int8, device=a.device)
    if out.dtype != torch.int8 or tuple(out.shape) != (m, n) or out.stride(1) != 1 or out.device != a.device:
        raise ShapeError("requant: out must be int8 [M, N] with unit column stride on A's device")
    check(_lib.load().ngemm_cuda_gemm_u8i8_requant(
        a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), out.data_ptr(), out.stride(0), m, n, k,
        scale.data_ptr(), bias.data_ptr() if bias is not None else None, int(zero_point), int(mode),
        _stream_ptr(stream)))
    return out


def gemm_device_batched(a, b, c=None, mode: SatMode = SatMode.WIDENING_EXACT, stream=None):
    """C[z] = A[z] * B[z]^T for a batch of GEMMs of one shape, on CUDA torch tensors.

    A: uint8 [G, M, K] (or [M, K], broadcast), B: int8 [G, N, K] (or [N, K]), C: int32 [G, M, N].
    Skinny shapes (M <= 16) run as one launch over the whole batch (ngemm_cuda_gemm_u8i8_strided_batched).
    """
    import torch
    if a.dtype != torch.uint8 or b.dtype != torch.int8:
        raise UnsupportedError(f"gemm: no kernel path for {a.dtype} x {b.dtype}")
    if a.dim() not in (2, 3) or b.dim() not in (2, 3) or a.shape[-1] != b.shape[-1]:
        raise ShapeError(f"batched gemm: A is {tuple(a.shape)}, B is {tuple(b.shape)}")
    if a.stride(-1) != 1 or b.stride(-1) != 1:
        raise ShapeError("gemm: operands must be K-contiguous")
    g = a.shape[0] if a.dim() == 3 else (b.shape[0] if b.dim() == 3 else 1)
    if (a.dim() == 3 and a.shape[0] != g) or (b.dim() == 3 and b.shape[0] != g):
        raise ShapeError("batched gemm: batch sizes of A and B differ")
    m, k = a.shape[-2], a.shape[-1]
    n = b.shape[-2]
    sa = a.stride(0) if a.dim() == 3 else 0
    sb = b.stride(0) if b.dim() == 3 else 0
    if c is None:
        c = torch.empty((g, m, n), dtype=torch.int32, device=a.device)
    if c.dtype != torch.int32 or tuple(c.shape) != (g, m, n) or c.stride(2) != 1:
        raise ShapeError("batched gemm: C must be int32 [G, M, N] with unit column stride")
    check(_lib.load().ngemm_cuda_gemm_u8i8_strided_batched(
        a.data_ptr(), a.stride(-2), sa, b.data_ptr(), b.stride(-2), sb, c.data_ptr(), c.stride(1), c.stride(0),
        g, m, n, k, int(mode), _stream_ptr(stream)))
    return c


class DevicePackedWeight:
    """Device-resident prepacked weight (opaque ngemm_packed_handle)."""

    def __init__(self, handle):
        self.h = handle

    @classmethod
    def from_packed(cls, p: PackedWeight) -> "DevicePackedWeight":
        h = C.c_void_p()
        data = np.ascontiguousarray(p.data)
        meta = p.meta()
        check(_lib.load().ngemm_cuda_packed_upload(C.byref(meta), data.ctypes.data, data.nbytes, C.byref(h)))
        return cls(h)

    @classmethod
    def from_device(cls, a) -> "DevicePackedWeight":
        h = C.c_void_p()
        check(_lib.load().ngemm_cuda_packed_from_device(a.data_ptr(), a.stride(0), a.shape[0], a.shape[1],
                                                          C.byref(h)))
        return cls(h)

    def info(self):
        d_a, lda, m, k, dev = C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
        check(_lib.load().ngemm_cuda_packed_info(self.h, C.byref(d_a), C.byref(lda), C.byref(m), C.byref(k),
                                                   C.byref(dev)))
        return d_a.value, lda.value, m.value, k.value, dev.value

    def gemm(self, b, c=None, mode: SatMode = SatMode.WIDENING_EXACT, stream=None):
        import torch
        _, _, m, k, _ = self.info()
        n = b.shape[0]
        if b.dtype != torch.int8 or b.shape[1] != k or b.stride(1) != 1:
            raise ShapeError(f"gemm_packed: packed K={k} but B is {tuple(b.shape)}")
        if c is None:
            c = torch.empty((m, n), dtype=torch.int32, device=b.device)
        check(_lib.load().ngemm_cuda_gemm_packed(self.h, b.data_ptr(), b.stride(0), c.data_ptr(), c.stride(0), n,
                                                   int(mode), _stream_ptr(stream)))
        return c

    def free(self):
        if self.h:
            _lib.load().ngemm_cuda_packed_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def repack_device(p: PackedWeight, d_packed, d_a, lda: int, stream=None):
    """Device repack of packed bytes (torch uint8 tensor) into row-major A (torch uint8 [M, lda])."""
    meta = p.meta()
    check(_lib.load().ngemm_cuda_repack(C.byref(meta), d_packed.data_ptr(), d_a.data_ptr(), lda,
                                          _stream_ptr(stream)))


def pick_kernel(m, n, k, mode) -> str:
    return _lib.KERNEL_NAMES[_lib.load().ngemm_cuda_pick_kernel(m, n, k, int(mode))]


def shard_rows(m: int, ndev: int, align: int = 128):
    """Row blocks of the M-shard driver (contiguous, tile-aligned): list of ndev+1 boundaries."""
    out = (C.c_int64 * (ndev + 1))()
    check(_lib.load().ngemm_cuda_shard_rows(m, ndev, align, out))
    return list(out)


def gemm_multi(devices, a: np.ndarray, b: np.ndarray, mode: SatMode, gather_device: int = -1):
    """Single-process M-shard over `devices` (host arrays), B replicated, no collective.
    Returns C on the host; with gather_device >= 0 also returns the device pointer of the
    full C assembled on that device by peer copies (free with ngemm_cuda_free)."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    _check_operands(a, b)
    m, k = a.shape
    n = b.shape[0]
    c = np.empty((m, n), np.int32)
    devs = (C.c_int * len(devices))(*devices)
    g = C.c_void_p()
    check(_lib.load().ngemm_cuda_gemm_u8i8_multi(devs, len(devices), a.ctypes.data, b.ctypes.data, c.ctypes.data,
                                                   m, n, k, int(mode), gather_device,
                                                   C.byref(g) if gather_device >= 0 else None))
    return (c, g.value) if gather_device >= 0 else c


class ShardedPackedWeight:
    """A packed weight split by rows over several GPUs and kept resident there (whole tm-strips
    per device; ngemm_cuda_packed_upload_sharded)."""

    def __init__(self, p: PackedWeight, devices):
        self.devices = list(devices)
        self.m, self.k = p.m_orig, p.k_orig
        data = np.ascontiguousarray(p.data)
        meta = p.meta()
        devs = (C.c_int * len(self.devices))(*self.devices)
        self.h = (C.c_void_p * len(self.devices))()
        check(_lib.load().ngemm_cuda_packed_upload_sharded(C.byref(meta), data.ctypes.data, data.nbytes, devs,
                                                             len(self.devices), self.h))

    def gemm(self, b: np.ndarray, mode: SatMode) -> np.ndarray:
        """gemm_ngemm on the sharded weight: host B in, host C out (B replicated over NVLink)."""
        b = np.ascontiguousarray(b)
        if b.dtype != np.int8 or b.ndim != 2 or b.shape[1] != self.k:
            raise ShapeError(f"sharded gemm: B must be int8 [N, {self.k}]")
        c = np.empty((self.m, b.shape[0]), np.int32)
        check(_lib.load().ngemm_cuda_gemm_packed_multi(self.h, len(self.devices), b.ctypes.data, c.ctypes.data,
                                                         b.shape[0], int(mode)))
        return c

    def free(self):
        L = _lib.load()
        for i in range(len(self.devices)):
            if self.h[i]:
                L.ngemm_cuda_packed_free(self.h[i])
                self.h[i] = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def tune(m: int, n: int, k: int, mode: SatMode, repeats: int = 5, warmup: int = 2) -> dict:
    """GPU autotuner (the reference's tune(), tuner.hpp:132-175, re-targeted): every applicable
    kernel configuration is verified bit-for-bit against the CUDA-core reference kernel, then
    timed (median of `repeats` after `warmup`); the winner becomes the dispatcher's choice for
    this shape in this process.  Raises TuneError if a candidate mis-computes."""
    rec = _lib.TuneRecord()
    check(_lib.load().ngemm_cuda_tune(m, n, k, int(mode), repeats, warmup, C.byref(rec)))
    return {f: getattr(rec, f) for f, _ in rec._fields_}


def tune_store_save(path: str):
    check(_lib.load().ngemm_cuda_tune_store_save(path.encode()))


def tune_store_load(path: str) -> int:
    n = C.c_int()
    check(_lib.load().ngemm_cuda_tune_store_load(path.encode(), C.byref(n)))
    return n.value


def tune_clear():
    check(_lib.load().ngemm_cuda_tune_clear())


__all__ = [
    "SatMode", "Engine", "Perm", "KernelShape", "kernel_shape", "TileConfig", "PackedWeight", "pack_weights",
    "unpack_weights", "gemm_conventional", "gemm_ngemm", "gemm_device", "DevicePackedWeight", "repack_device",
    "pick_kernel", "shard_rows", "gemm_multi", "NgemmError", "ShapeError", "UnsupportedError", "ConfigError",
    "RangeError", "CorruptionError", "IndexError_", "CudaError", "TuneError", "tune", "tune_store_save",
    "tune_store_load", "tune_clear",
]

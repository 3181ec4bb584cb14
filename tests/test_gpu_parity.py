"""GPU parity: every kernel of libngemm_cuda.so, called through the C-ABI, is bit-exact
against the CPU oracle (pinned to the reference) and the reference-generated fixtures.

Modes: SAT = HardwareSaturating (gemm_sat_oracle, gemm.hpp:83-104), EXACT = WideningExact
(gemm_ref, gemm.hpp:36-52).  Integer work: the bar is bit-exact, no tolerance."""
import ctypes
import os

import numpy as np
import pytest

from oracle.oracle import EXACT, SAT
from paper_1910_00178_b200 import _lib, api

pytestmark = pytest.mark.gpu

KERNELS = {"simt": _lib.KERNEL_SIMT, "tcgen05": _lib.KERNEL_TCGEN05, "skinny": _lib.KERNEL_SKINNY,
           "sat_hybrid": _lib.KERNEL_SAT_HYBRID, "auto": _lib.KERNEL_AUTO}


def dev_gemm(a, b, mode, kernel="auto", lda=None, ldb=None, ldc=None):
    import torch
    m, k = a.shape
    n = b.shape[0]
    lda = k if lda is None else lda
    ldb = k if ldb is None else ldb
    ldc = n if ldc is None else ldc
    da = torch.zeros((m, lda), dtype=torch.uint8, device="cuda")
    db = torch.zeros((n, ldb), dtype=torch.int8, device="cuda")
    da[:, :k] = torch.from_numpy(a)
    db[:, :k] = torch.from_numpy(b)
    # C lives inside a canary frame: 8 sentinel rows before and after, and sentinel padding
    # columns when ldc > n — any store outside the logical [m x n] block is caught (the pool's
    # compute-sanitizer is closed, so out-of-bounds writes are checked this way)
    frame = torch.full((m + 16, ldc), 0x5A5A5A5A, dtype=torch.int32, device="cuda")
    dc = frame[8:8 + m]
    L = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(L.ngemm_cuda_gemm_u8i8_ex(da.data_ptr(), lda, db.data_ptr(), ldb, dc.data_ptr(), ldc, m, n, k, mode,
                                         KERNELS[kernel], st))
    torch.cuda.synchronize()
    full = frame.cpu().numpy()
    assert (full[:8] == 0x5A5A5A5A).all() and (full[8 + m:] == 0x5A5A5A5A).all(), "kernel wrote outside C's rows"
    out = full[8:8 + m]
    if ldc > n:
        assert (out[:, n:] == 0x5A5A5A5A).all(), "kernel wrote outside C's logical columns"
    return out[:, :n]


def kernels_for(m, mode):
    ks = ["simt", "auto"]
    if mode == EXACT:
        ks.append("tcgen05")
    if m <= 16:
        ks.append("skinny")
    return ks


def test_2x2(cuda):
    a = np.array([[1, 2], [3, 4]], np.uint8)
    b = np.array([[5, -1], [2, 0]], np.int8)
    for mode in (EXACT, SAT):
        for k in kernels_for(2, mode):
            assert dev_gemm(a, b, mode, k).tolist() == [[3, 2], [11, 6]], k


def test_adversarial_saturation(cuda, golden):
    adv = golden["adversarial"]
    a = np.full((4, 12), 255, np.uint8)
    b = np.array(adv["b"], np.int8)
    for k in kernels_for(4, SAT):
        assert dev_gemm(a, b, SAT, k).tolist() == adv["sat"], k
    for k in kernels_for(4, EXACT):
        assert dev_gemm(a, b, EXACT, k).tolist() == adv["exact"], k


def test_random_small_shapes_vs_reference(cuda, oracle, golden):
    for case in golden["random_small"]:
        a = oracle.mat_random_u8(case["m"], case["k"], case["seed_a"])
        b = oracle.mat_random_i8(case["n"], case["k"], case["seed_b"])
        for mode, key in ((EXACT, "exact"), (SAT, "sat")):
            for k in kernels_for(case["m"], mode):
                assert dev_gemm(a, b, mode, k).ravel().tolist() == case[key], (case["m"], case["n"], case["k"], k)


@pytest.mark.parametrize("seed", range(4))
def test_random_shapes_1_to_300(cuda, oracle, seed):
    rng = np.random.default_rng(seed)
    for _ in range(12):
        m, n, k = (int(x) for x in rng.integers(1, 300, 3))
        a = oracle.mat_random_u8(m, k, 10 * seed + m)
        b = oracle.mat_random_i8(n, k, 10 * seed + n + 7)
        for mode in (EXACT, SAT):
            ref = oracle.gemm(a, b, mode)
            for kern in kernels_for(m, mode):
                assert (dev_gemm(a, b, mode, kern) == ref).all(), (m, n, k, mode, kern)


def test_acceptance_1000_random_small(cuda, oracle):
    # SPEC.md:533 acceptance #1: >= 1000 random (M,N,K) in [1,64]^3, exact mode, bit-exact
    rng = np.random.default_rng(1234)
    for t in range(1000):
        m, n, k = (int(x) for x in rng.integers(1, 65, 3))
        a = oracle.mat_random_u8(m, k, 5000 + t)
        b = oracle.mat_random_i8(n, k, 9000 + t)
        assert (dev_gemm(a, b, EXACT) == oracle.gemm(a, b, EXACT, threads=1)).all(), (m, n, k)


def test_acceptance_100_adversarial_sat(cuda, oracle):
    # SPEC.md:534 acceptance #2: 100 adversarial cases (u8 = 255, i8 in {127, -128})
    rng = np.random.default_rng(99)
    for t in range(100):
        m, n, k = (int(x) for x in rng.integers(1, 65, 3))
        a = np.full((m, k), 255, np.uint8)
        b = np.where(rng.integers(0, 2, (n, k)) == 1, 127, -128).astype(np.int8)
        ref = oracle.gemm(a, b, SAT, threads=1)
        for kern in kernels_for(m, SAT):
            assert (dev_gemm(a, b, SAT, kern) == ref).all(), (m, n, k, kern)


def test_wrapping_k4096(cuda, oracle):
    a = oracle.mat_random_u8(2, 4096, 30)
    b = oracle.mat_random_i8(2, 4096, 31)
    for mode in (EXACT, SAT):
        ref = oracle.gemm(a, b, mode)
        for kern in kernels_for(2, mode) + (["tcgen05"] if mode == EXACT else []):
            assert (dev_gemm(a, b, mode, kern) == ref).all(), kern


def test_leading_dimensions_and_unaligned_k(cuda, oracle):
    for (m, n, k, lda, ldb, ldc) in ((130, 70, 1000, 1003, 1001, 77), (17, 300, 37, 40, 48, 301),
                                     (5, 33, 100, 100, 112, 33), (300, 260, 200, 208, 200, 264)):
        a = oracle.mat_random_u8(m, k, m)
        b = oracle.mat_random_i8(n, k, n)
        for mode in (EXACT, SAT):
            ref = oracle.gemm(a, b, mode)
            for kern in kernels_for(m, mode):
                assert (dev_gemm(a, b, mode, kern, lda, ldb, ldc) == ref).all(), (m, n, k, kern)


def test_config1(cuda, oracle, golden):
    a = oracle.mat_random_u8(1024, 1024, 0)
    b = oracle.mat_random_i8(1024, 1024, 1)
    g = golden["config1"]
    for mode, key in ((EXACT, "exact"), (SAT, "sat")):
        for kern in kernels_for(1024, mode):
            c = dev_gemm(a, b, mode, kern)
            assert oracle.fnv1a(c) == g[f"{key}_fnv"], kern
            assert int(c.astype(np.int64).sum()) == g[f"{key}_checksum"]


def test_config2_skinny(cuda, oracle, golden):
    for c in golden["config2"]:
        a = oracle.mat_random_u8(c["m"], c["k"], 0)
        b = oracle.mat_normal_i8(c["n"], c["k"], 1, 32.0)
        for mode, key in ((EXACT, "exact"), (SAT, "sat")):
            for kern in kernels_for(c["m"], mode):
                assert oracle.fnv1a(dev_gemm(a, b, mode, kern)) == c[f"{key}_fnv"], (c["m"], c["n"], c["k"], kern)


def test_config3_medium(cuda, oracle, golden):
    for c in golden["config3"]:
        a = oracle.mat_random_u8(c["m"], c["k"], 0)
        b = oracle.mat_random_i8(c["n"], c["k"], 1)
        for mode, key in ((EXACT, "exact"), (SAT, "sat")):
            for kern in kernels_for(c["m"], mode):
                assert oracle.fnv1a(dev_gemm(a, b, mode, kern)) == c[f"{key}_fnv"], (c["m"], c["n"], c["k"], kern)


def _pattern(kind, rows, cols, p):
    idx = np.arange(rows * cols).reshape(rows, cols) & 1
    if kind == "a":
        return np.full((rows, cols), 255, np.uint8) if p == "all255" else np.where(idx, 255, 0).astype(np.uint8)
    if p == "all-128":
        return np.full((rows, cols), -128, np.int8)
    if p == "all127":
        return np.full((rows, cols), 127, np.int8)
    return np.where(idx, 127, -128).astype(np.int8)


def test_config4_saturation_edges(cuda, golden):
    for c in golden["config4"]:
        s = c["size"]
        a = _pattern("a", s, s, c["a"])
        b = _pattern("b", s, s, c["b"])
        for mode, key in ((EXACT, "exact"), (SAT, "sat")):
            for kern in kernels_for(s, mode):
                out = dev_gemm(a, b, mode, kern)
                assert (out == c[key]).all(), (s, c["a"], c["b"], key, kern)


def test_splitk_small_m_deep_k(cuda, oracle):
    # few output tiles and deep K: exercises the split-K (red.add) epilogue of tcgen05
    for (m, n, k) in ((128, 256, 8192), (200, 100, 4000), (64, 64, 16384)):
        a = oracle.mat_random_u8(m, k, 1)
        b = oracle.mat_random_i8(n, k, 2)
        assert (dev_gemm(a, b, EXACT, "tcgen05") == oracle.gemm(a, b, EXACT)).all(), (m, n, k)


def test_packed_path_device(cuda, oracle):
    import torch
    for (m, n, k, tm, tn, tk, perm, w, v) in ((9, 3, 7, 8, 2, 4, 0, 32, 8), (40, 17, 100, 16, 8, 12, 3, 32, 8),
                                              (300, 129, 520, 32, 64, 64, 4, 64, 16),
                                              (130, 257, 257, 16, 64, 260, 5, 64, 16)):
        a = oracle.mat_random_u8(m, k, m + 1)
        b = oracle.mat_random_i8(n, k, n + 1)
        p = api.pack_weights(a, api.KernelShape(w, 4, v), api.TileConfig(tm, tn, tk, api.Perm(perm)))
        dp = p.upload()
        _, lda, mm, kk, _ = dp.info()
        assert (mm, kk) == (m, k) and lda % 16 == 0
        db = torch.from_numpy(b).cuda()
        for mode in (EXACT, SAT):
            c = dp.gemm(db, mode=mode).cpu().numpy()
            assert (c == oracle.gemm(a, b, mode)).all(), (m, n, k, perm, mode)
        # device repack entry on its own
        dpk = torch.from_numpy(p.data).cuda()
        da = torch.zeros((m, lda), dtype=torch.uint8, device="cuda")
        api.repack_device(p, dpk, da, lda)
        torch.cuda.synchronize()
        assert (da[:, :k].cpu().numpy() == a).all()
        p.invalidate()


def test_host_api_mirrors_reference_tests(cuda, oracle, golden):
    s256 = api.kernel_shape(256)
    # test_gemm.cpp:73-79, 101-107
    a = np.array([[1, 2], [3, 4]], np.uint8)
    b = np.array([[5, -1], [2, 0]], np.int8)
    for eng in (api.Engine.AUTO, api.Engine.EMULATED, api.Engine.CUDA):
        assert api.gemm_conventional(a, b, s256, api.SatMode.WIDENING_EXACT, eng).tolist() == [[3, 2], [11, 6]]
        p = api.pack_weights(a, s256, api.TileConfig(8, 1, 4))
        assert api.gemm_ngemm(p, b, api.SatMode.WIDENING_EXACT, eng).tolist() == [[3, 2], [11, 6]]
    # test_gemm.cpp:109-116: zero weights through the padding path
    z = api.gemm_ngemm(api.pack_weights(np.zeros((9, 5), np.uint8), s256, api.TileConfig(8, 1, 4)),
                       oracle.mat_random_i8(4, 5, 6), api.SatMode.HARDWARE_SATURATING, api.Engine.EMULATED)
    assert (z == 0).all()
    # test_gemm.cpp:118-127: tail stress across permutations, both modes
    a = oracle.mat_random_u8(9, 7, 12, 0, 127)
    b = oracle.mat_random_i8(3, 7, 13)
    ref = oracle.gemm(a, b, EXACT)
    for perm in (api.Perm.MNK, api.Perm.NMK, api.Perm.KNM):
        p = api.pack_weights(a, s256, api.TileConfig(8, 2, 4, perm))
        for mode in api.SatMode:
            assert (api.gemm_ngemm(p, b, mode, api.Engine.EMULATED) == ref).all()
            assert (api.gemm_ngemm(p, b, mode) == ref).all()
    # reference-kernel digests on packed weights (emulated reference, both modes)
    for c in golden["ngemm_packed"]:
        a = oracle.mat_random_u8(c["m"], c["k"], c["seed_a"])
        b = oracle.mat_random_i8(c["n"], c["k"], c["seed_b"])
        p = api.pack_weights(a, s256, api.TileConfig(c["tm"], c["tn"], c["tk"], api.Perm(c["perm"])))
        assert oracle.fnv1a(api.gemm_ngemm(p, b, api.SatMode.WIDENING_EXACT)) == c["exact_fnv"]
        assert oracle.fnv1a(api.gemm_ngemm(p, b, api.SatMode.HARDWARE_SATURATING)) == c["sat_fnv"]
    with pytest.raises(api.UnsupportedError):
        api.gemm_conventional(a, b, s256, api.SatMode.WIDENING_EXACT, api.Engine.NATIVE)


def test_multi_device_driver_single_gpu(cuda, oracle):
    a = oracle.mat_random_u8(300, 200, 3)
    b = oracle.mat_random_i8(150, 200, 4)
    for mode in (EXACT, SAT):
        assert (api.gemm_multi([0], a, b, mode) == oracle.gemm(a, b, mode)).all()
        # same device listed twice = two row shards on one GPU (host-side shard/concat logic)
        assert (api.gemm_multi([0, 0], a, b, mode) == oracle.gemm(a, b, mode)).all()
        # gather of the row shards into one device buffer (peer copies; here device 0 -> 0)
        import ctypes
        import glob
        import nvidia.cuda_runtime
        rt = ctypes.CDLL(glob.glob(os.path.join(list(nvidia.cuda_runtime.__path__)[0], "lib", "libcudart.so*"))[0])
        rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
        c, ptr = api.gemm_multi([0, 0], a, b, mode, gather_device=0)
        full = np.empty_like(c)
        assert rt.cudaMemcpy(full.ctypes.data, ptr, full.nbytes, 2) == 0  # cudaMemcpyDeviceToHost
        assert (full == c).all() and (c == oracle.gemm(a, b, mode)).all()
        _lib.check(_lib.load().ngemm_cuda_free(ptr))


def _c5_row_blocks(m, block=64, count=8, seed=5):
    """Row blocks of C checked against the oracle: the first and the last row tile plus random
    64-row blocks in between (seeded), sorted, non-overlapping starts."""
    rng = np.random.default_rng(seed)
    starts = {0, m - block}
    while len(starts) < count:
        starts.add(int(rng.integers(1, (m - block) // block)) * block)
    return sorted(starts)


def test_multi_device_driver_pipeline_and_sharded_weight(cuda, oracle):
    """The multi-GPU entries on one GPU listed several times (each listing = one row shard; the
    NVLink relay of B becomes device-local copies): B copied once and relayed, A rows streamed in
    and C rows out through the host pipeline (pageable and pinned), the peer-copy gather, and
    the sharded resident weight for every permutation (M-before-K shards are plain byte ranges,
    K-before-M shards are gathered per K tile row)."""
    import torch
    for (m, n, k) in [(1000, 900, 333), (3000, 4100, 1024)]:
        a = oracle.mat_random_u8(m, k, 41)
        b = oracle.mat_random_i8(n, k, 42)
        for mode in (EXACT, SAT):
            ref = oracle.gemm(a, b, mode)
            assert (api.gemm_multi([0, 0, 0], a, b, mode) == ref).all(), (m, n, k, mode)
            ta, tb = torch.from_numpy(a).pin_memory(), torch.from_numpy(b).pin_memory()
            tc = torch.full((m, n), -1, dtype=torch.int32).pin_memory()
            devs = (ctypes.c_int * 4)(0, 0, 0, 0)
            _lib.check(_lib.load().ngemm_cuda_gemm_u8i8_multi(devs, 4, ta.data_ptr(), tb.data_ptr(), tc.data_ptr(),
                                                              m, n, k, mode, -1, None))
            assert (tc.numpy() == ref).all(), ("pinned", m, n, k, mode)
    a = oracle.mat_random_u8(1500, 640, 43)
    b = oracle.mat_random_i8(700, 640, 44)
    for perm in range(6):
        p = api.pack_weights(a, api.KernelShape(64, 4, 16), api.TileConfig(32, 64, 64, api.Perm(perm)))
        for devs in ([0], [0, 0], [0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]):  # the last: more devices than blocks
            w = api.ShardedPackedWeight(p, devs)
            try:
                for mode in (EXACT, SAT):
                    assert (w.gemm(b, mode) == oracle.gemm(a, b, mode)).all(), (perm, len(devs), mode)
            finally:
                w.free()


@pytest.mark.slow
@pytest.mark.parametrize("mode", [EXACT, SAT])
def test_config5_full_size(cuda, oracle, golden, mode):
    """16384^3 (config 5) through AUTO in both modes — exact runs the tcgen05 pair kernel,
    HardwareSaturating the tensor-core + sparse-fix chain (64 K-chunks per row, 128 MiB of
    index lists):
      * rows 0-127 against the reference's own digest and checksum (golden, oracle/_ref),
      * 8 row blocks of 64 rows (first and last row tile + 6 random) bit-exact against the
        oracle (gemm_ref / gemm_sat_oracle restated, gemm.hpp:36-52, 83-104),
      * exact mode: 16 Freivalds rounds over the WHOLE C, C.x == A.(B^T.x) with x in [0, 16)
        in float64 — exact, since |C| < 2^30 (no wrap at K = 16384) and every partial sum is an
        integer below 16384 * 255 * 128 * 16 * 16384 < 2^53.  A single wrong element escapes
        one round with probability <= 1/16, all 16 with <= 2^-64."""
    import torch
    K = 16384
    b = oracle.mat_random_i8(K, K, 1)
    g = golden["config5_rows0_128"]
    assert oracle.fnv1a(b) == golden["config5_b_fnv"]
    a = oracle.mat_random_u8(K, K, 0)
    da = torch.from_numpy(a).cuda()
    db = torch.from_numpy(b).cuda()
    assert _lib.load().ngemm_cuda_pick_kernel(K, K, K, mode) == (
        _lib.KERNEL_TCGEN05 if mode == EXACT else _lib.KERNEL_SAT_HYBRID)
    dc = api.gemm_device(da, db, mode=mode)
    torch.cuda.synchronize()
    key = "exact" if mode == EXACT else "sat"
    top = dc[:128].cpu().numpy()
    assert oracle.fnv1a(top) == g[f"{key}_fnv"]
    assert int(top.astype(np.int64).sum()) == g[f"{key}_checksum"]
    for r0 in _c5_row_blocks(K):
        got = dc[r0:r0 + 64].cpu().numpy()
        ref = oracle.gemm(np.ascontiguousarray(a[r0:r0 + 64]), b, mode)
        assert (got == ref).all(), (key, r0, int((got != ref).sum()))
    if mode == EXACT:
        gen = torch.Generator(device="cuda").manual_seed(7)
        x = torch.randint(0, 16, (K, 16), device="cuda", generator=gen).to(torch.float64)
        lhs = dc.to(torch.float64) @ x                      # C.x, 16 rounds at once
        btx = db.to(torch.float64).t() @ x                  # B^T x
        rhs = da.to(torch.float64) @ btx                    # A.(B^T x)
        assert torch.equal(lhs, rhs)


def test_dispatcher_fuzz_auto(cuda, oracle):
    """AUTO dispatch over 160 seeded random problems drawn around every planner boundary (skinny
    M <= 16 with narrow / wide N and shallow / deep K, the saturating MMA + fix kernel's M > 8,
    cluster and atomic K splits, 1-CTA / pair / split-K tcgen05 shapes, the SIMT / hybrid size
    rule), ragged sizes and padded leading dimensions, both SatModes, weight-like and uniform B —
    every result bit-exact against the oracle."""
    rng = np.random.default_rng(20251021)
    def pick(lo, hi):
        return int(np.exp(rng.uniform(np.log(lo), np.log(hi))))
    for it in range(160):
        kind = it % 4
        if kind == 0:    # skinny
            m, n, k = int(rng.integers(1, 17)), pick(1, 6000), pick(1, 20000)
        elif kind == 1:  # small / medium
            m, n, k = pick(17, 700), pick(1, 1500), pick(1, 3000)
        elif kind == 2:  # wide or deep
            m, n, k = pick(17, 300), pick(500, 5000), pick(500, 9000)
        else:            # around the hybrid's size rule (M >= 256, >= 1e9 MACs)
            m, n, k = pick(200, 1200), pick(700, 1500), pick(700, 1500)
        while 2.0 * m * n * k > 6e9:
            k = max(1, k // 2)
        pad = int(rng.integers(0, 3))
        lda = k + (0 if pad == 0 else int(rng.integers(1, 40)))
        ldb = k + (0 if pad == 0 else int(rng.integers(1, 40)))
        ldc = n + (0 if pad != 2 else int(rng.integers(1, 9)))
        a = oracle.mat_random_u8(m, k, 1000 + it)
        b = oracle.mat_normal_i8(n, k, 2000 + it, 32.0) if it % 3 else oracle.mat_random_i8(n, k, 2000 + it)
        for mode in (EXACT, SAT):
            got = dev_gemm(a, b, mode, "auto", lda, ldb, ldc)
            assert (got == oracle.gemm(a, b, mode)).all(), (it, m, n, k, lda, ldb, ldc, mode)


@pytest.mark.slow
def test_pair512_tiles_through_auto_ragged(cuda, oracle):
    """A ragged deep-K problem that AUTO runs on the 256 x 512 pair tiles (K >= 8192, >= 4 waves):
    4100 x 8300 x 8200, partial tiles on M and N, a K tail inside a 128-byte slab, padded ldc.  Eight row
    blocks (first / last tile rows and random ones) bit-exact against the oracle, and 16 Freivalds
    rounds over the whole C (exact in float64: |C| < 2^31, x < 16, sums < 2^53)."""
    import torch
    m, n, k = 4100, 8300, 8200
    a = oracle.mat_random_u8(m, k, 31)
    b = oracle.mat_random_i8(n, k, 32)
    da = torch.zeros((m, 8208), dtype=torch.uint8, device="cuda")
    db = torch.zeros((n, 8208), dtype=torch.int8, device="cuda")
    da[:, :k] = torch.from_numpy(a)
    db[:, :k] = torch.from_numpy(b)
    frame = torch.full((m, 8304), 0x5A5A5A5A, dtype=torch.int32, device="cuda")
    dc = frame[:, :n]
    api.gemm_device(da[:, :k], db[:, :k], dc, mode=EXACT)
    torch.cuda.synchronize()
    assert (frame[:, n:] == 0x5A5A5A5A).all()
    for r0 in (0, 192, 2048 - 32, 4100 - 64, 1000, 3333, 3840, 4032):
        got = dc[r0:r0 + 64].cpu().numpy()
        assert (got == oracle.gemm(np.ascontiguousarray(a[r0:r0 + 64]), b, EXACT)).all(), r0
    gen = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randint(0, 16, (n, 16), device="cuda", generator=gen).to(torch.float64)
    lhs = dc.to(torch.float64) @ x
    rhs = da[:, :k].to(torch.float64) @ (db[:, :k].to(torch.float64).t() @ x)
    assert torch.equal(lhs, rhs)


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4, 5, 6, 7, 8, 9])
def test_tcgen05_every_tile_config_and_split(cuda, oracle, cfg, knobs):
    """Each tcgen05 tile configuration (pair 256x256, 1-CTA 128x256/128/64, the 4-CTA and 2-CTA
    A-multicast clusters, the lean 2-3 stage variants), with and without
    split-K (TMA s32 reduce-add), with TMA-store and direct-store epilogues, vs the oracle."""
    knobs.set("TC_CFG", str(cfg))
    for splits, direct in (("1", "0"), ("1", "1"), ("2", "0"), ("3", "0")):
        knobs.set("TC_SPLITS", splits)
        knobs.set("TC_DIRECT", direct)  # TMA-store vs direct vector-store epilogue
        # (300, 333, 777, 336): ldc % 4 == 0 but N % 4 != 0 — must not take the TMA epilogue (a box
        # straddling the last column writes the whole trailing 16-byte granule, probe_ldc.py)
        for (m, n, k, ldc) in ((300, 520, 1100, None), (256, 256, 2048, 260), (129, 65, 640, None),
                               (513, 300, 1024, 301), (600, 1024, 700, None), (256, 512, 128, 516),
                               (300, 333, 777, 336)):
            a = oracle.mat_random_u8(m, k, m + cfg)
            b = oracle.mat_random_i8(n, k, n + cfg)
            got = dev_gemm(a, b, EXACT, "tcgen05", ldc=ldc)
            assert (got == oracle.gemm(a, b, EXACT)).all(), (cfg, splits, direct, m, n, k, ldc)


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_tcgen05_tail_split(cuda, oracle, cfg, knobs):
    """Tail split (TileMap::full_tiles): when the last wave of tiles would leave more than half the
    SMs idle, its tiles run as two half-width work items (N = BN/2 MMAs, half-height B boxes, half
    the epilogue).  Shapes whose tile counts trigger it for every tile configuration, ragged ones
    included (a half tile straddling N), bit-exact against the oracle, and the same with the split
    switched off; plus the fused-requant epilogue on a split shape."""
    import torch
    knobs.set("TC_CFG", cfg)
    shapes = [(4096, 1280, 640), (4000, 1250, 333), (2048, 2560, 384), (1000, 9000, 256)]
    for (m, n, k) in shapes:
        a = oracle.mat_random_u8(m, k, m + 7)
        b = oracle.mat_random_i8(n, k, n + 7)
        ref = oracle.gemm(a, b, EXACT)
        for sched in (1, 0):
            knobs.set("TC_SCHED", sched)
            got = dev_gemm(a, b, EXACT, "tcgen05")
            assert (got == ref).all(), (cfg, sched, m, n, k, int((got != ref).sum()))
    knobs.set("TC_SCHED", 1)
    m, n, k = 4096, 1280, 640
    a = oracle.mat_random_u8(m, k, 3)
    b = oracle.mat_random_i8(n, k, 4)
    scale = np.linspace(1e-4, 3e-3, n).astype(np.float32)
    bias = np.arange(n, dtype=np.int32) * 37 - 20000
    out = api.gemm_device_requant(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                                  torch.from_numpy(scale).cuda(), torch.from_numpy(bias).cuda(), zero_point=3)
    torch.cuda.synchronize()
    y = requant_ref(oracle.gemm(a, b, EXACT), scale, bias, 3)
    assert (out.cpu().numpy() == y).all(), int((out.cpu().numpy() != y).sum())


@pytest.mark.parametrize("variant", ["0", "1", "2", "3", "4", "5"])
def test_skinny_variants(cuda, oracle, golden, variant, knobs):
    """Skinny (M <= 16) variants: 0 warp-butterfly dp4a, 1 lanes-own-rows dp4a (broadcast A),
    2 tensor-core swap-AB, 3 warp-MMA load stream (2 and 3: exact mode only; sat falls back
    to 1), 4 dp4a load stream (sat), 5 warp-MMA + sparse fix (sat; exact falls back to 1) — all
    bit-exact."""
    knobs.set("SKINNY_VARIANT", variant)
    for c in golden["config2"]:
        a = oracle.mat_random_u8(c["m"], c["k"], 0)
        b = oracle.mat_normal_i8(c["n"], c["k"], 1, 32.0)
        for mode, key in ((EXACT, "exact"), (SAT, "sat")):
            assert oracle.fnv1a(dev_gemm(a, b, mode, "skinny")) == c[f"{key}_fnv"], (variant, c["m"], c["n"], c["k"])
    for (m, n, k, lda, ldb, ldc) in ((3, 1000, 1000, 1000, 1000, 1000), (16, 129, 4097, 4112, 4100, 131),
                                     (7, 70, 33, 40, 48, 70), (1, 5000, 160, 160, 160, 5003), (16, 300, 12288, None, None, None)):
        a = oracle.mat_random_u8(m, k, m)
        b = oracle.mat_random_i8(n, k, n)
        for mode in (EXACT, SAT):
            assert (dev_gemm(a, b, mode, "skinny", lda, ldb, ldc) == oracle.gemm(a, b, mode)).all(), (variant, m, n, k)


def test_skinny_cluster_k_splits(cuda, oracle, knobs):
    """Grid K splits of the skinny load streams (exact warp-MMA stream, saturating MMA + fix): two
    splits (up to 8 with SKINNY_XRED=2) form a thread-block cluster and meet through distributed
    shared memory (no zeroed C, no atomics); more splits, or SKINNY_XRED=0, wrap-add into a zeroed C.  Deep-K / narrow-N
    shapes where the planner splits on its own, and forced split counts, ragged K included."""
    for (m, n, k, lda, ldb, ldc) in ((16, 768, 3072, None, None, None), (16, 48, 16384, None, None, None),
                                     (9, 256, 16384, None, None, None), (16, 130, 4097, 4112, 4100, 131),
                                     (5, 64, 1000, None, None, None)):
        a = oracle.mat_random_u8(m, k, m + 21)
        b = oracle.mat_normal_i8(n, k, n + 22, 32.0)
        for mode in (EXACT, SAT):
            ref = oracle.gemm(a, b, mode)
            for xred in ("2", "1", "0"):  # 2: clusters for up to 8 splits, 1: default (two splits), 0: never
                knobs.set("SKINNY_XRED", xred)
                for splits in ("-1", "2", "3", "5", "8", "11"):
                    knobs.set("SKINNY_SPLITS", splits)
                    got = dev_gemm(a, b, mode, "skinny", lda, ldb, ldc)
                    assert (got == ref).all(), (m, n, k, mode, xred, splits, int((got != ref).sum()))
    knobs.set("SKINNY_VARIANT", "5")  # the MMA + fix stream for M <= 8 too
    a = oracle.mat_random_u8(7, 2048, 3)
    b = oracle.mat_normal_i8(96, 2048, 4, 32.0)
    for splits in ("2", "4"):
        knobs.set("SKINNY_SPLITS", splits)
        assert (dev_gemm(a, b, SAT, "skinny") == oracle.gemm(a, b, SAT)).all(), splits


def test_skinny_sat_tensor_core_fix(cuda, oracle, knobs):
    """skinny_sathyb_kernel (variant 5): exact warp MMAs plus the sparse correction of the pairs
    with |b0 + b1| >= 129, and its dense branch (> 128 listed words per warp chunk).  Threshold
    pairs (64,65), (65,64), (-64,-65), (64,64), (127,-128), saturated pairs (127,127),
    (-128,-128) sprinkled into a weight-like B (sparse branch), uniform and all-extreme B (dense
    branch), A all 255 / alternating / uniform, ragged K and N, unaligned leading dimensions, K
    splits over the grid, 8 and 16 warps."""
    import numpy as np
    knobs.set("SKINNY_VARIANT", "5")
    rng = np.random.default_rng(11)
    special = np.array([[64, 65], [65, 64], [-64, -65], [-65, -64], [64, 64], [-64, -64], [127, -128], [-128, 127],
                        [127, 127], [-128, -128], [127, 2], [-128, -1], [0, 127], [-128, 0], [100, 29], [-100, -29]], np.int8)
    shapes = [(16, 4096, 1024, None, None, None), (9, 768, 3072, None, None, None), (16, 130, 1001, 1008, 1003, 132),
              (5, 77, 255, None, None, None), (16, 48, 16384, None, None, None), (12, 3072, 768, None, None, None),
              (8, 1000, 130, 144, 131, 1000), (16, 16, 127, None, None, None), (3, 4096, 1024, None, None, None)]
    for (m, n, k, lda, ldb, ldc) in shapes:
        for bkind in ("normal", "uniform", "max", "min", "alt"):
            if bkind == "normal":
                b = oracle.mat_normal_i8(n, k, n + 5, 32.0).copy()
                # sprinkle threshold / saturating pairs at even-aligned positions
                for _ in range(max(4, n * k // 2000)):
                    r, j = int(rng.integers(0, n)), int(rng.integers(0, max(1, k // 2)))
                    if 2 * j + 1 < k:
                        b[r, 2 * j:2 * j + 2] = special[int(rng.integers(0, len(special)))]
            elif bkind == "uniform":
                b = oracle.mat_random_i8(n, k, n + 6)
            else:
                b = np.full((n, k), 127 if bkind == "max" else -128, np.int8)
                if bkind == "alt":
                    b[:, 1::2] = 127
            for akind in ("uniform", "max", "alt"):
                if akind == "uniform":
                    a = oracle.mat_random_u8(m, k, m + 3)
                else:
                    a = np.full((m, k), 255, np.uint8)
                    if akind == "alt":
                        a[:, 0::2] = 0
                ref = oracle.gemm(a, b, SAT)
                for warps in ("-1", "8", "16"):
                    knobs.set("SKINNY_WARPS", warps)
                    got = dev_gemm(a, b, SAT, "skinny", lda, ldb, ldc)
                    assert (got == ref).all(), (m, n, k, bkind, akind, warps, int((got != ref).sum()))
                knobs.set("SKINNY_WARPS", "-1")
                knobs.set("SKINNY_SPLITS", "3")
                got = dev_gemm(a, b, SAT, "skinny", lda, ldb, ldc)
                knobs.set("SKINNY_SPLITS", "-1")
                assert (got == ref).all(), (m, n, k, bkind, akind, "splits", int((got != ref).sum()))


@pytest.mark.parametrize("hybrid", ["1", "-1"])
def test_sat_mode_on_provably_safe_inputs(cuda, oracle, hybrid, knobs):
    """HardwareSaturating on inputs that cannot saturate (the reference's safe range, u8 <= 127,
    tuner.hpp:26-43): with max A measured on the device no pair is classified as clampable, so
    the tensor cores compute everything and the fix kernel exits; the result must still equal
    gemm_sat_oracle (== gemm_ref here).  Also the boundary cases around max A = 128 / 129.
    hybrid=1 forces the tensor-core chain on every shape, -1 is the default dispatch."""
    knobs.set("SAT_HYBRID", hybrid)
    for (m, n, k) in ((512, 512, 1024), (1000, 700, 333), (2048, 2048, 2048)):
        a = oracle.mat_random_u8(m, k, 3, 0, 127)
        b = oracle.mat_random_i8(n, k, 4)
        got = dev_gemm(a, b, SAT, "auto")
        assert (got == oracle.gemm(a, b, SAT)).all() and (got == oracle.gemm(a, b, EXACT)).all()
    # 2*amax*bmax = 2*128*127 = 32512 <= 32767 but 2*amax*bneg = 2*128*128 = 32768: still safe
    a = np.full((300, 256), 128, np.uint8)
    b = np.where(np.arange(200 * 256).reshape(200, 256) % 3 == 0, -128, 127).astype(np.int8)
    assert (dev_gemm(a, b, SAT, "auto") == oracle.gemm(a, b, SAT)).all()
    # one byte over the edge: 129 * 127 * 2 = 32766 ok, 129 * 128 * 2 = 33024 saturates
    a[7, 10] = 129
    a[7, 11] = 129
    b[:, 10] = -128
    b[:, 11] = -128
    got = dev_gemm(a, b, SAT, "auto")
    assert (got == oracle.gemm(a, b, SAT)).all()
    assert (got != oracle.gemm(a, b, EXACT)).any()


def _normal_i8(rng, shape, sigma=32.0):
    return np.clip(np.rint(rng.normal(0.0, sigma, shape)), -128, 127).astype(np.int8)


@pytest.mark.parametrize("case", ["uniform", "normal", "extreme", "dense_frac", "sparse_edges", "safe_b"])
def test_sat_hybrid_tensor_core_plus_fix(cuda, oracle, case, knobs):
    """HardwareSaturating for M > 16 (kernel_satfix.cuh): tcgen05 on B with the pairs that could
    clamp zeroed, plus the CUDA-core fix of those pairs (list walk, or the list-free path for rows
    whose pairs all could clamp).  Sparse, dense and empty lists, ragged shapes (odd K, K < 256, K
    not a multiple of 16, unaligned leading dimensions) must equal gemm_sat_oracle bit for bit."""
    rng = np.random.default_rng(["uniform", "normal", "extreme", "dense_frac", "sparse_edges", "safe_b"].index(case))
    # NGEMM_SAT_HYBRID=1 forces the chain below its size threshold (M >= 256, >= 1e9 MACs);
    # 1000^3 takes it by default
    knobs.set("SAT_HYBRID", "1")
    # N % 4 != 0 (333) cannot take the TMA reduce-add: AUTO falls back to the CUDA-core kernel
    # (260, 256, 40000): 157 K chunks > the fix kernel's 128-chunk list, so K is split on the host
    shapes = [(300, 332, 777), (300, 333, 777), (257, 388, 200), (40, 640, 1024), (129, 4100, 100),
              (1000, 1000, 1000), (512, 1280, 1024), (260, 256, 40000)]
    for (m, n, k) in shapes:
        a = rng.integers(0, 256, (m, k), dtype=np.uint8)
        if case == "uniform":
            b = rng.integers(-128, 128, (n, k), dtype=np.int8)
        elif case == "normal":
            b = _normal_i8(rng, (n, k))
        elif case == "extreme":
            a[:] = 255
            b = np.full((n, k), 127, np.int8)
            b[::3] = -128
        elif case == "dense_frac":  # ~70 % of the pairs can clamp: long lists, some full rows
            b = np.where(rng.random((n, k)) < 0.84, 127, rng.integers(-128, 128, (n, k))).astype(np.int8)
        elif case == "sparse_edges":  # a few dangerous pairs at chunk edges and in the odd-K tail
            b = rng.integers(-50, 51, (n, k), dtype=np.int8)
            for (r, c) in ((0, 0), (n - 1, k - 1), (n // 2, min(254, k - 1)), (n // 2, min(255, k - 1)),
                           (n // 3, min(256, k - 1)), (1, k - 2)):
                b[r, c] = 127 if (r + c) % 2 else -128
                b[r, c ^ 1 if (c ^ 1) < k else c] = 127 if (r + c) % 2 else -128
        else:  # safe_b: no pair can clamp although A spans [0, 255]
            b = rng.integers(-64, 65, (n, k), dtype=np.int8)
        ref = oracle.gemm(a, b, SAT)
        got = dev_gemm(a, b, SAT, "auto")
        assert (got == ref).all(), (case, m, n, k, int((got != ref).sum()))
        if (m, n, k) in ((300, 332, 777), (300, 333, 777)):  # ragged leading dimensions (no 16-byte loads)
            got = dev_gemm(a, b, SAT, "auto", lda=k + 3, ldb=k + 5, ldc=n + 4 - n % 4)  # ldc % 4 == 0
            assert (got == ref).all(), (case, "ld", int((got != ref).sum()))


def test_sat_hybrid_explicit_kernel_id(cuda, oracle):
    """NGEMM_KERNEL_SAT_HYBRID chosen explicitly: bit-exact on a small shape (below the AUTO size
    rule); refused for exact mode, M <= 16 and a C that TMA cannot describe."""
    a = oracle.mat_random_u8(100, 300, 5)
    b = oracle.mat_random_i8(200, 300, 6)
    assert (dev_gemm(a, b, SAT, "sat_hybrid") == oracle.gemm(a, b, SAT)).all()
    for (aa, bb, mode, ldc) in ((a, b, EXACT, None), (a[:16], b, SAT, None), (a, b, SAT, 201),
                                (a, b[:199], SAT, 200)):  # N % 4 != 0
        with pytest.raises(_lib.UnsupportedError):
            dev_gemm(aa, bb, mode, "sat_hybrid", ldc=ldc)


@pytest.mark.parametrize("hybrid", ["0", "1"])
def test_host_entry_pipelined_pinned(cuda, oracle, hybrid, knobs):
    """ngemm_cuda_gemm_u8i8_host on PINNED host buffers takes the chunked H2D/compute/D2H
    pipeline (C >= 64 MiB); result must equal the oracle in both modes.  hybrid=1 forces the
    saturating tensor-core chain on every C tile (strided C sub-blocks, ragged tiles)."""
    import torch
    knobs.set("SAT_HYBRID", hybrid)
    L = _lib.load()
    # 4096^2 splits into 8 x 4 C tiles; 4000 x 4500 x 333 gives ragged row/column tiles and padded K
    for (m, n, k) in [(4096, 4096, 640), (4000, 4500, 333)]:
        a = oracle.mat_random_u8(m, k, 11)
        b = oracle.mat_random_i8(n, k, 12)
        ta = torch.from_numpy(a).pin_memory()
        tb = torch.from_numpy(b).pin_memory()
        tc = torch.empty((m, n), dtype=torch.int32).pin_memory()
        for mode in (EXACT, SAT):
            tc.fill_(-1)
            _lib.check(L.ngemm_cuda_gemm_u8i8_host(ta.data_ptr(), tb.data_ptr(), tc.data_ptr(), m, n, k, mode, 0))
            assert (tc.numpy() == oracle.gemm(a, b, mode)).all(), (m, n, k, mode)


@pytest.mark.parametrize("pinning", ["none", "a_only", "c_only"])
def test_host_entry_pipelined_pageable_staging(cuda, oracle, pinning):
    """The host pipeline on PAGEABLE buffers (what gemm_conventional on std::vector-backed
    MatrixBufs passes): operands and C move through the pinned staging ring, copied by the host
    worker pool; mixed pinned / pageable operands take the direct copy for the pinned ones.
    Ragged tiles, K not a multiple of 16, growing row blocks, a C tile wider than one slot."""
    import torch
    L = _lib.load()
    for (m, n, k) in [(4000, 4500, 333), (2304, 4000, 4100), (6000, 2048, 64)]:
        a = oracle.mat_random_u8(m, k, 21)
        b = oracle.mat_random_i8(n, k, 22)
        c = np.full((m, n), -1, np.int32)
        if pinning == "a_only":
            ta = torch.from_numpy(a).pin_memory()
            a_ptr, b_ptr, c_ptr, out = ta.data_ptr(), b.ctypes.data, c.ctypes.data, c
        elif pinning == "c_only":
            tc = torch.from_numpy(c).pin_memory()
            a_ptr, b_ptr, c_ptr, out = a.ctypes.data, b.ctypes.data, tc.data_ptr(), None
        else:
            a_ptr, b_ptr, c_ptr, out = a.ctypes.data, b.ctypes.data, c.ctypes.data, c
        for mode in (EXACT, SAT):
            _lib.check(L.ngemm_cuda_gemm_u8i8_host(a_ptr, b_ptr, c_ptr, m, n, k, mode, 0))
            got = out if out is not None else tc.numpy()
            assert (got == oracle.gemm(a, b, mode)).all(), (pinning, m, n, k, mode)


@pytest.mark.parametrize("pinned", [True, False])
def test_resident_weight_host_pipeline(cuda, oracle, pinned):
    """gemm_ngemm's path: the weight A resident in HBM (packed handle), B streamed in by column
    blocks and C tiles streamed out (ngemm_cuda_gemm_packed_resident_host), pinned or pageable."""
    import ctypes as C
    import torch
    L = _lib.load()
    for (m, n, k) in [(3000, 5000, 777), (1024, 8192, 128)]:
        a = oracle.mat_random_u8(m, k, 31)
        b = oracle.mat_random_i8(n, k, 32)
        da = torch.from_numpy(a).cuda()
        h = C.c_void_p()
        _lib.check(L.ngemm_cuda_packed_from_device(da.data_ptr(), k, m, k, C.byref(h)))
        try:
            for mode in (EXACT, SAT):
                if pinned:
                    tb = torch.from_numpy(b).pin_memory()
                    tc = torch.full((m, n), -1, dtype=torch.int32).pin_memory()
                    _lib.check(L.ngemm_cuda_gemm_packed_resident_host(h, tb.data_ptr(), tc.data_ptr(), n, mode))
                    got = tc.numpy()
                else:
                    got = np.full((m, n), -1, np.int32)
                    _lib.check(L.ngemm_cuda_gemm_packed_resident_host(h, b.ctypes.data, got.ctypes.data, n, mode))
                assert (got == oracle.gemm(a, b, mode)).all(), (pinned, m, n, k, mode)
        finally:
            L.ngemm_cuda_packed_free(h)


def test_autotuner_picks_verified_config_and_dispatch_stays_exact(cuda, oracle, tmp_path):
    """GPU autotuner (tuner.hpp:132-175 re-targeted): the record names a configuration that was
    verified against the reference kernel; afterwards the dispatcher uses it and results stay
    bit-exact; the store round-trips."""
    api.tune_clear()
    for (m, n, k, mode) in ((512, 1024, 1024, EXACT), (16, 4096, 1024, EXACT), (300, 700, 520, SAT),
                            (4, 768, 3072, SAT)):
        rec = api.tune(m, n, k, mode, repeats=3, warmup=1)
        assert rec["m"] == m and rec["median_ns"] > 0 and rec["min_ns"] <= rec["median_ns"]
        assert rec["kernel"] in (0, 1, 2, 3)
        a = oracle.mat_random_u8(m, k, 21)
        b = oracle.mat_random_i8(n, k, 22)
        assert (dev_gemm(a, b, mode, "auto") == oracle.gemm(a, b, mode)).all(), rec
    path = tmp_path / "store.txt"
    api.tune_store_save(str(path))
    api.tune_clear()
    assert api.tune_store_load(str(path)) == 4
    api.tune_clear()


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,k", [(1, 768, 768), (4, 1000, 333), (16, 4096, 1024), (9, 257, 4096), (64, 300, 200)])
def test_strided_batched(cuda, oracle, m, n, k):
    """ngemm_cuda_gemm_u8i8_strided_batched: every batch member equals its own reference GEMM;
    padded strides between members and between C slices are never written."""
    import torch
    g = 5
    lda, ldb, ldc = k + 16, k + 32, n + 8
    sa, sb, sc = m * lda + 48, n * ldb + 16, m * ldc + 40
    rng = np.random.default_rng(m * 7 + n)
    a = rng.integers(0, 256, size=g * sa, dtype=np.uint8)
    b = rng.integers(-128, 128, size=g * sb, dtype=np.int8)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    L = _lib.load()
    for mode in (0, 1):
        dc = torch.full((g * sc,), 0x5A5A5A5A, dtype=torch.int32, device="cuda")
        _lib.check(L.ngemm_cuda_gemm_u8i8_strided_batched(da.data_ptr(), lda, sa, db.data_ptr(), ldb, sb,
                                                          dc.data_ptr(), ldc, sc, g, m, n, k, mode,
                                                          torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        c = dc.cpu().numpy()
        written = np.zeros(g * sc, bool)
        for z in range(g):
            az = a[z * sa: z * sa + m * lda].reshape(m, lda)[:, :k]
            bz = b[z * sb: z * sb + n * ldb].reshape(n, ldb)[:, :k]
            cz = c[z * sc: z * sc + m * ldc].reshape(m, ldc)[:, :n]
            assert (cz == oracle.gemm(np.ascontiguousarray(az), np.ascontiguousarray(bz), mode)).all(), (z, mode)
            idx = z * sc + np.arange(m)[:, None] * ldc + np.arange(n)[None, :]
            written[idx.ravel()] = True
        assert (c[~written] == 0x5A5A5A5A).all(), "batched kernel wrote outside a C slice"


@pytest.mark.gpu
def test_batched_broadcast_and_api(cuda, oracle):
    import torch
    rng = np.random.default_rng(3)
    a = rng.integers(0, 256, size=(8, 4096), dtype=np.uint8)
    b = rng.integers(-128, 128, size=(6, 1024, 4096), dtype=np.int8)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    for mode in (api.SatMode.HARDWARE_SATURATING, api.SatMode.WIDENING_EXACT):
        c = api.gemm_device_batched(da, db, mode=mode).cpu().numpy()  # A broadcast (stride 0)
        for z in range(6):
            assert (c[z] == oracle.gemm(a, b[z], int(mode))).all()
    with pytest.raises(api.ShapeError):
        api.gemm_device_batched(torch.zeros((2, 4, 8), dtype=torch.uint8, device="cuda"),
                                torch.zeros((3, 4, 8), dtype=torch.int8, device="cuda"))


def _dev_gemm_i16(a, b):
    import torch
    m, k = a.shape
    n = b.shape[0]
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    frame = torch.full((m + 16, n), 0x5A5A5A5A, dtype=torch.int32, device="cuda")
    L = _lib.load()
    _lib.check(L.ngemm_cuda_gemm_i16(da.data_ptr(), k, db.data_ptr(), k, frame[8:8 + m].data_ptr(), n, m, n, k,
                                     torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    full = frame.cpu().numpy()
    assert (full[:8] == 0x5A5A5A5A).all() and (full[8 + m:] == 0x5A5A5A5A).all(), "i16 kernel wrote outside C"
    return full[8:8 + m]


@pytest.mark.gpu
@pytest.mark.parametrize("path", ["simt", "tcgen05"])
def test_i16_paths_vs_reference_golden(cuda, oracle, golden, path, knobs):
    """i16 x i16 (gemm.hpp:161-190): the CUDA-core kernel and the tensor-core byte-plane
    decomposition (4 int8 tcgen05 GEMMs, shifted and reduce-added) against the reference."""
    knobs.set("I16_PATH", path)
    for c in golden["i16"]:
        a = oracle.mat_random_i16(c["m"], c["k"], c["seed"], c["lo"], c["hi"])
        b = oracle.mat_random_i16(c["n"], c["k"], c["seed"] + 100, c["lo"], c["hi"])
        out = _dev_gemm_i16(a, b)
        assert oracle.fnv1a(out) == c["c_fnv"], (path, c)
    rng = np.random.default_rng(11)
    for (m, n, k) in [(300, 129, 777), (17, 64, 16), (256, 512, 4096), (1000, 1000, 1000)]:
        a = rng.integers(-32768, 32768, size=(m, k), dtype=np.int16)
        b = rng.integers(-32768, 32768, size=(n, k), dtype=np.int16)
        assert (_dev_gemm_i16(a, b) == oracle.gemm_i16(a, b)).all(), (path, m, n, k)


@pytest.mark.gpu
def test_i16_byte_planes_on_pair512_tiles(cuda, oracle, knobs):
    """The i16 byte-plane decomposition (shifted stores / TMA reduce-adds of four int8 GEMMs) forced
    onto the 256 x 512 pair tiles, which AUTO takes for large i16 problems with deep K."""
    knobs.set("I16_PATH", "tcgen05")
    knobs.set("TC_CFG", 9)
    rng = np.random.default_rng(12)
    for (m, n, k) in [(300, 1100, 512), (513, 520, 777)]:
        a = rng.integers(-32768, 32768, size=(m, k), dtype=np.int16)
        b = rng.integers(-32768, 32768, size=(n, k), dtype=np.int16)
        assert (_dev_gemm_i16(a, b) == oracle.gemm_i16(a, b)).all(), (m, n, k)


def requant_ref(c, scale, bias, zp):
    """The fused requantisation's arithmetic in numpy (ngemm_cuda.h): int32 + bias wraps,
    float32 round-to-nearest conversion, one fp32 multiply, rint (half to even), clamp."""
    acc = c.astype(np.int64) + (bias.astype(np.int64) if bias is not None else 0)
    acc = ((acc + 2**31) % 2**32 - 2**31).astype(np.int32)
    prod = np.clip(acc.astype(np.float32) * scale.astype(np.float32), np.float32(-1e6), np.float32(1e6))
    return np.clip(np.rint(prod).astype(np.int64) + zp, -128, 127).astype(np.int8)


@pytest.mark.parametrize("mode", [EXACT, SAT])
def test_fused_requant_epilogue(cuda, oracle, mode):
    """ngemm_cuda_gemm_u8i8_requant: exact mode requantises in the kernel epilogue (tcgen05 for
    M > 16, the warp-MMA stream for M <= 16; int32 C never stored); the saturating mode goes
    through C in scratch + requant_kernel.
    Bit-exact against the numpy statement of the same arithmetic, per-column scales spanning the
    clamp edges, with and without bias, several zero points, ragged N and output pitch."""
    import torch
    rng = np.random.default_rng(5 + mode)
    for (m, n, k, ldo, zp, with_bias) in ((300, 333, 777, 340, 0, True), (2048, 1024, 1024, None, -3, False),
                                          (16, 4096, 1024, None, 7, True), (129, 64, 640, 67, 0, True),
                                          (257, 512, 2048, None, 1, True), (1, 768, 768, 770, 2, True),
                                          (5, 333, 1001, None, 0, False)):
        a = oracle.mat_random_u8(m, k, m)
        b = oracle.mat_random_i8(n, k, n)
        scale = (rng.uniform(1.0 / 4000.0, 1.0 / 1000.0, n)).astype(np.float32)
        bias = rng.integers(-200000, 200000, n, dtype=np.int32) if with_bias else None
        ref = requant_ref(oracle.gemm(a, b, mode), scale, bias, zp)
        ldo = n if ldo is None else ldo
        dev = torch.device("cuda")
        out = torch.full((m, ldo), 0x55, dtype=torch.int8, device=dev)[:, :n]
        got = api.gemm_device_requant(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev),
                                      torch.from_numpy(scale).to(dev),
                                      torch.from_numpy(bias).to(dev) if bias is not None else None, zp, out=out,
                                      mode=mode)
        torch.cuda.synchronize()
        full = got.cpu().numpy()
        assert (full == ref).all(), (mode, m, n, k, int((full != ref).sum()))
        assert (ref == 127).any() and (ref == -128).any(), "the case should exercise both clamp edges"
        pad = out.as_strided((m, ldo), (ldo, 1)).cpu().numpy()[:, n:]
        assert (pad == 0x55).all(), "requant wrote outside the logical columns"


def test_fused_requant_epilogue_pair512_tiles(cuda, oracle, knobs):
    """The requantising epilogue on the 256 x 512 pair tiles (TC_CFG 9, the configuration AUTO
    takes for deep K and many waves): TMEM column -> tile column permutation, ragged M / N and a
    padded output pitch."""
    import torch
    knobs.set("TC_CFG", 9)
    rng = np.random.default_rng(17)
    for (m, n, k, ldo, zp) in ((300, 1100, 1024, 1104, -2), (513, 512, 384, None, 0)):
        a = oracle.mat_random_u8(m, k, m + 40)
        b = oracle.mat_random_i8(n, k, n + 41)
        scale = (rng.uniform(1.0 / 4000.0, 1.0 / 1000.0, n)).astype(np.float32)
        bias = rng.integers(-200000, 200000, n, dtype=np.int32)
        ref = requant_ref(oracle.gemm(a, b, EXACT), scale, bias, zp)
        ldo = n if ldo is None else ldo
        out = torch.full((m, ldo), 0x55, dtype=torch.int8, device="cuda")[:, :n]
        got = api.gemm_device_requant(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
                                      torch.from_numpy(scale).cuda(), torch.from_numpy(bias).cuda(), zp, out=out)
        torch.cuda.synchronize()
        assert (got.cpu().numpy() == ref).all(), (m, n, k)
        pad = out.as_strided((m, ldo), (ldo, 1)).cpu().numpy()[:, n:]
        assert (pad == 0x55).all(), "requant wrote outside the logical columns"


def test_stress_repeated_launches_across_streams(cuda, oracle, knobs):
    """Race / sync stress (compute-sanitizer is closed on this pool): the warp-specialised
    mbarrier/TMEM pipelines, the cluster DSMEM reduction, split-K TMA reduce-add and the
    saturating chain are launched many times back to back on 4 concurrent streams, with
    different grids per shape, each launch into its own C.  Every output must equal the
    oracle bit for bit — a missing fence, barrier phase slip or TMEM/smem reuse race shows up
    as a sporadic mismatch."""
    import torch
    cases = [  # (m, n, k, mode, kernel, knob settings)
        (2048, 2048, 2048, EXACT, "tcgen05", {}),                            # pair 256x256, persistent
        (300, 520, 1100, EXACT, "tcgen05", {"TC_CFG": 2, "TC_SPLITS": 3}),   # 1-CTA + split-K reduce-add
        (600, 1024, 700, EXACT, "tcgen05", {"TC_CFG": 4}),                   # 4-CTA A-multicast clusters
        (16, 4096, 1024, EXACT, "skinny", {}),                               # warp-MMA load stream
        (16, 4096, 1024, EXACT, "skinny", {"SKINNY_VARIANT": 2}),            # tcgen05 swap-AB, DSMEM split-K
        (16, 4096, 1024, SAT, "skinny", {}),                                 # dp4a load stream
        (1000, 1000, 1000, SAT, "auto", {}),                                 # tensor cores + sparse fix
    ]
    streams = [torch.cuda.Stream() for _ in range(4)]
    reps = 24
    for (m, n, k, mode, kern, kv) in cases:
        for name, v in kv.items():
            knobs.set(name, v)
        a = oracle.mat_random_u8(m, k, m + 1)
        b = oracle.mat_random_i8(n, k, n + 2)
        ref = oracle.gemm(a, b, mode)
        da = torch.from_numpy(a).cuda()
        db = torch.from_numpy(b).cuda()
        outs = [torch.full((m, n), 0x5A5A5A5A, dtype=torch.int32, device="cuda") for _ in range(reps)]
        torch.cuda.synchronize()
        for i in range(reps):
            s = streams[i % len(streams)]
            with torch.cuda.stream(s):
                api.gemm_device(da, db, outs[i], mode=mode, kernel=KERNELS[kern], stream=s)
        torch.cuda.synchronize()
        for i, o in enumerate(outs):
            got = o.cpu().numpy()
            assert (got == ref).all(), (m, n, k, mode, kern, kv, i, int((got != ref).sum()))
        _lib.reset_options()

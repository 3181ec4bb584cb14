"""Generate tests/golden/golden.json from the UNMODIFIED reference (oracle/_ref).

Run here, where /root/reference exists (`make -C oracle` builds oracle/_ref first):
    python tests/golden/make_golden.py
Every number in the fixture is produced by the reference's own functions (mat_random,
gemm_ref, gemm_sat_oracle, gemm_conventional, gemm_ngemm, pack_weights) through
oracle/ref_shim.cpp — never by our oracle restatement, which the tests then pin against it.
The c2 normal-B generator is ours; its draws come from oracle/liboracle.so.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import EXACT, SAT, Oracle, Reference  # noqa: E402

U8, I8 = 0, 1


def fnv(arr):
    h = 1469598103934665603
    for byte in np.ascontiguousarray(arr).view(np.uint8).tobytes():
        h ^= byte
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def main():
    ref = Reference()
    ora = Oracle()
    fast_fnv = ora.fnv1a  # byte digest only (pure hashing, cross-checked with fnv() below)
    g = {"generator": "tests/golden/make_golden.py via oracle/_ref (unmodified reference)",
         "host_isa_bits": ref.host_isa_bits()}

    # --- PRNG goldens (test_matrix.cpp:37-59)
    g["mat_random_i8_1x4_seed1_m3_3"] = ref.mat_random(I8, 1, 4, 1, -3, 3).ravel().tolist()
    m64 = ref.mat_random(U8, 64, 64, 42, 0, 255)
    g["mat_random_u8_64x64_seed42_fnv"] = fnv(m64)
    assert fast_fnv(m64) == g["mat_random_u8_64x64_seed42_fnv"]
    g["mat_random_u8_16x16_seed0"] = ref.mat_random(U8, 16, 16, 0, 0, 255).ravel().tolist()
    g["mat_random_i8_16x16_seed1"] = ref.mat_random(I8, 16, 16, 1, -128, 127).ravel().astype(int).tolist()

    # --- 2x2 (test_gemm.cpp:44-52)
    a = np.array([[1, 2], [3, 4]], np.uint8)
    b = np.array([[5, -1], [2, 0]], np.int8)
    g["gemm_2x2"] = ref.gemm("gemm_ref", a, b).tolist()

    # --- adversarial saturation block (test_gemm.cpp:183-200): A=255, B = +127/-128 by rng(55)
    b = np.empty((3, 12), np.int8)
    draws = ref.mat_random(U8, 3, 12, 55, 0, 1)  # same stream as XorShift64Star(55).next_in(0, 1)
    b[:] = np.where(draws == 1, 127, -128)
    a = np.full((4, 12), 255, np.uint8)
    g["adversarial"] = {"b": b.astype(int).tolist(),
                        "sat": ref.gemm("gemm_sat_oracle", a, b).tolist(),
                        "exact": ref.gemm("gemm_ref", a, b).tolist(),
                        "conv_sat_emulated": ref.gemm("gemm_conventional", a, b, SAT, engine=1, isa_bits=256).tolist()}

    # --- randomized small shapes (test_gemm.cpp:213-229 style, full range, both modes)
    rs = []
    rng_draws = ref.mat_random(U8, 1, 180, 77, 0, 255).ravel()
    for t in range(60):
        m = 1 + int(rng_draws[3 * t]) % 24
        n = 1 + int(rng_draws[3 * t + 1]) % 24
        k = 1 + int(rng_draws[3 * t + 2]) % 40
        A = ref.mat_random(U8, m, k, 1000 + t, 0, 255)
        B = ref.mat_random(I8, n, k, 2000 + t, -128, 127)
        rs.append({"m": m, "n": n, "k": k, "seed_a": 1000 + t, "seed_b": 2000 + t,
                   "exact": ref.gemm("gemm_ref", A, B).ravel().tolist(),
                   "sat": ref.gemm("gemm_sat_oracle", A, B).ravel().tolist()})
    g["random_small"] = rs

    # --- packing byte layouts (test_layout.cpp:61-146) and random configs
    packs = []
    for (m, k, w, h, v, tm, tn, tk, perm, seed) in [
        (2, 2, 32, 4, 8, 8, 1, 4, 0, None), (16, 8, 32, 4, 8, 8, 1, 4, 0, 11), (16, 8, 32, 4, 8, 8, 1, 4, 5, 11),
        (16, 8, 32, 4, 8, 16, 1, 8, 0, 11), (37, 101, 32, 4, 8, 8, 1, 4, 0, 5), (19, 23, 32, 4, 8, 16, 4, 8, 2, 8),
        (33, 70, 64, 4, 16, 32, 64, 12, 3, 9), (100, 64, 16, 4, 4, 8, 1, 16, 4, 10), (5, 5, 32, 4, 8, 8, 1, 4, 0, 3),
        (130, 257, 64, 4, 16, 16, 64, 260, 0, 12),
    ]:
        A = np.array([[1, 2], [3, 4]], np.uint8) if seed is None else ref.mat_random(U8, m, k, seed, 0, 255)
        P = ref.pack(A, w, h, v, tm, tn, tk, perm)
        packs.append({"m": m, "k": k, "w": w, "h": h, "v": v, "tm": tm, "tn": tn, "tk": tk, "perm": perm,
                      "seed": seed, "nbytes": int(P.size), "fnv": fnv(P),
                      "head": P[:64].tolist()})
    g["packs"] = packs

    # --- gemm_ngemm through the reference kernels on packed weights (emulated, both modes)
    ng = []
    for (m, n, k, tm, tn, tk, perm) in [(9, 3, 7, 8, 2, 4, 0), (9, 3, 7, 8, 2, 4, 2), (9, 3, 7, 8, 2, 4, 5),
                                        (40, 17, 100, 16, 8, 12, 3), (64, 64, 256, 32, 64, 64, 4)]:
        A = ref.mat_random(U8, m, k, 300 + m, 0, 255)
        B = ref.mat_random(I8, n, k, 400 + n, -128, 127)
        P = ref.pack(A, 32, 4, 8, tm, tn, tk, perm)
        meta = ora.packed_meta(m, k, 32, 4, 8, tm, tn, tk, perm)
        ng.append({"m": m, "n": n, "k": k, "tm": tm, "tn": tn, "tk": tk, "perm": perm,
                   "seed_a": 300 + m, "seed_b": 400 + n,
                   "exact_fnv": fnv(ref.gemm_ngemm_packed(P, meta, B, EXACT, engine=1)),
                   "sat_fnv": fnv(ref.gemm_ngemm_packed(P, meta, B, SAT, engine=1))})
    g["ngemm_packed"] = ng

    # --- config 4: pattern x shape known answers, both modes
    def pattern(kind, rows, cols, p):
        if kind == U8:
            if p == "all255":
                return np.full((rows, cols), 255, np.uint8)
            return np.where(np.arange(rows * cols).reshape(rows, cols) & 1, 255, 0).astype(np.uint8)
        if p == "all-128":
            return np.full((rows, cols), -128, np.int8)
        if p == "all127":
            return np.full((rows, cols), 127, np.int8)
        return np.where(np.arange(rows * cols).reshape(rows, cols) & 1, 127, -128).astype(np.int8)

    c4 = []
    for s in (2048, 1000):
        for pa in ("all255", "alt0_255"):
            for pb in ("all-128", "all127", "alt-128_127"):
                # every C element is equal: one row of A against all of B is enough for the reference
                A = pattern(U8, 1, s, pa)
                B = pattern(I8, s, s, pb)
                ce = ref.gemm("gemm_ref", A, B)
                cs = ref.gemm("gemm_sat_oracle", A, B)
                assert (ce == ce[0, 0]).all() and (cs == cs[0, 0]).all()
                c4.append({"size": s, "a": pa, "b": pb, "exact": int(ce[0, 0]), "sat": int(cs[0, 0])})
    g["config4"] = c4

    # --- i16 x i16 (gemm_ref and the emulated 16-bit gemm_conventional, gemm.hpp:161-190):
    # inputs from the reference's own mat_random(I16); the extreme case wraps mod 2^32
    i16 = []
    for (m, n, k, seed, lo, hi) in [(1, 1, 1, 3, -32768, 32767), (7, 5, 3, 4, -32768, 32767),
                                    (33, 17, 129, 5, -32768, 32767), (64, 48, 96, 6, -300, 300),
                                    (5, 9, 4096, 7, -32768, -32768), (40, 24, 1000, 8, -32768, 32767)]:
        a16 = ref.mat_random(2, m, k, seed, lo, hi)
        b16 = ref.mat_random(2, n, k, seed + 100, lo, hi)
        c_ref = ref.gemm_i16("gemm_ref", a16, b16)
        assert (ref.gemm_i16("gemm_conventional", a16, b16) == c_ref).all()
        i16.append({"m": m, "n": n, "k": k, "seed": seed, "lo": lo, "hi": hi, "a_fnv": fnv(a16),
                    "c_fnv": fnv(c_ref), "c_sum": int(c_ref.astype(np.int64).sum())})
    g["i16"] = i16

    # --- config 1 (1024^3, A seed 0 / B seed 1), both modes through the reference oracles
    t0 = time.time()
    A = ref.mat_random(U8, 1024, 1024, 0, 0, 255)
    B = ref.mat_random(I8, 1024, 1024, 1, -128, 127)
    ce = ref.gemm("gemm_ref", A, B)
    cs = ref.gemm("gemm_sat_oracle", A, B)
    g["config1"] = {"exact_checksum": int(ce.astype(np.int64).sum()), "sat_checksum": int(cs.astype(np.int64).sum()),
                    "exact_c00": int(ce[0, 0]), "sat_c00": int(cs[0, 0]), "exact_fnv": fast_fnv(ce),
                    "sat_fnv": fast_fnv(cs), "n_differ": int((ce != cs).sum())}
    print(f"config1 {time.time() - t0:.1f}s", flush=True)

    # --- config 3 (medium; uniform A seed 0, B seed 1): digests per shape and mode
    c3 = []
    for m in (128, 512, 2048):
        for (n, k) in ((1024, 1024), (4096, 1024), (1024, 4096)):
            A = ref.mat_random(U8, m, k, 0, 0, 255)
            B = ref.mat_random(I8, n, k, 1, -128, 127)
            se = ref.session(A, B, "gemm_ref", EXACT, threads=os.cpu_count())
            se.run()
            ce = se.result()
            ss = ref.session(A, B, "gemm_sat_oracle", SAT, threads=os.cpu_count())
            ss.run()
            cs = ss.result()
            c3.append({"m": m, "n": n, "k": k, "exact_fnv": fast_fnv(ce), "sat_fnv": fast_fnv(cs),
                       "exact_checksum": int(ce.astype(np.int64).sum()), "sat_checksum": int(cs.astype(np.int64).sum())})
            print(f"config3 {m}x{n}x{k} done {time.time() - t0:.1f}s", flush=True)
    g["config3"] = c3

    # --- config 2 (skinny; A uniform seed 0, B ~ N(0,32) clipped, our generator seed 1)
    c2 = []
    for m in (1, 4, 16):
        for (n, k) in ((768, 768), (3072, 768), (768, 3072), (4096, 1024)):
            A = ref.mat_random(U8, m, k, 0, 0, 255)
            B = ora.mat_normal_i8(n, k, 1, 32.0)
            ce = ref.gemm("gemm_ref", A, B)
            cs = ref.gemm("gemm_sat_oracle", A, B)
            c2.append({"m": m, "n": n, "k": k, "b_fnv": fast_fnv(B), "exact_fnv": fast_fnv(ce), "sat_fnv": fast_fnv(cs),
                       "n_differ": int((ce != cs).sum())})
    g["config2"] = c2

    # --- config 5 (16384^3): the first 128 rows of C through the reference (mat_random fills
    # row-major from one stream, so rows 0..127 of the seed-0 A are mat_random(U8,128,K,0)).
    A = ref.mat_random(U8, 128, 16384, 0, 0, 255)
    B = ref.mat_random(I8, 16384, 16384, 1, -128, 127)
    g["config5_b_fnv"] = fast_fnv(B)
    se = ref.session(A, B, "gemm_ref", EXACT, threads=os.cpu_count())
    se.run()
    ce = se.result()
    ss = ref.session(A, B, "gemm_sat_oracle", SAT, threads=os.cpu_count())
    ss.run()
    cs = ss.result()
    g["config5_rows0_128"] = {"exact_fnv": fast_fnv(ce), "sat_fnv": fast_fnv(cs),
                              "exact_checksum": int(ce.astype(np.int64).sum()),
                              "sat_checksum": int(cs.astype(np.int64).sum())}
    print(f"config5 rows done {time.time() - t0:.1f}s", flush=True)

    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(out, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", out)


if __name__ == "__main__":
    main()

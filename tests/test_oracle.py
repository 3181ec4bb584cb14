"""Pins the CPU oracle (oracle/oracle.c) against the reference's own golden vectors and
against fixtures produced by the unmodified reference (tests/golden/golden.json).
CPU only."""
import numpy as np
import pytest

from oracle.oracle import EXACT, SAT

U8, I8 = 0, 1


def test_prng_frozen_draws(oracle, golden):
    # test_matrix.cpp:37-50
    a = oracle.mat_random_i8(1, 4, 1, -3, 3)
    assert a.ravel().tolist() == [-2, -3, -3, -1]
    assert a.ravel().tolist() == golden["mat_random_i8_1x4_seed1_m3_3"]


def test_prng_golden_digest(oracle, golden):
    # test_matrix.cpp:52-59
    m = oracle.mat_random_u8(64, 64, 42)
    assert len(np.unique(m)) >= 200
    assert oracle.fnv1a(m) == 0x5D6A07D6EC6B5FFD == golden["mat_random_u8_64x64_seed42_fnv"]


def test_prng_streams_match_reference(oracle, golden):
    assert oracle.mat_random_u8(16, 16, 0).ravel().tolist() == golden["mat_random_u8_16x16_seed0"]
    assert oracle.mat_random_i8(16, 16, 1).ravel().tolist() == golden["mat_random_i8_16x16_seed1"]
    z = oracle.mat_random_u8(2, 2, 7, 0, 0)
    assert (z == 0).all()  # test_matrix.cpp:31-35


def test_gemm_2x2(oracle, golden):
    # test_gemm.cpp:44-52
    a = np.array([[1, 2], [3, 4]], np.uint8)
    b = np.array([[5, -1], [2, 0]], np.int8)
    for mode in (EXACT, SAT):
        assert oracle.gemm(a, b, mode).tolist() == [[3, 2], [11, 6]] == golden["gemm_2x2"]


def test_pair_semantics(oracle):
    # test_lanes.cpp:31-40 (saturation boundary) and 10-20 (basics)
    assert oracle.madd_pair(255, 255, 127, 127, SAT) == 32767
    assert oracle.madd_pair(255, 255, 127, 127, EXACT) == 64770
    assert oracle.madd_pair(255, 255, -128, -128, SAT) == -32768
    assert oracle.madd_pair(255, 255, -128, -128, EXACT) == -65280
    assert oracle.madd_pair(2, 3, 4, -1, SAT) == 5


def test_adversarial_saturation(oracle, golden):
    # test_gemm.cpp:183-200: A=255 against +-127/-128: sat != exact; oracle == reference
    adv = golden["adversarial"]
    a = np.full((4, 12), 255, np.uint8)
    b = np.array(adv["b"], np.int8)
    sat, exact = oracle.gemm(a, b, SAT), oracle.gemm(a, b, EXACT)
    assert (sat != exact).any()
    assert sat.tolist() == adv["sat"] == adv["conv_sat_emulated"]
    assert exact.tolist() == adv["exact"]


def test_zero_and_identity(oracle):
    # test_gemm.cpp:54-71
    a = oracle.mat_random_u8(5, 7, 1)
    assert (oracle.gemm(a, np.zeros((4, 7), np.int8), EXACT) == 0).all()
    eye = np.eye(6, dtype=np.uint8)
    b = oracle.mat_random_i8(4, 6, 9)
    for mode in (EXACT, SAT):
        assert (oracle.gemm(eye, b, mode) == b.T.astype(np.int32)).all()


def test_random_small_shapes_vs_reference(oracle, golden):
    for case in golden["random_small"]:
        a = oracle.mat_random_u8(case["m"], case["k"], case["seed_a"])
        b = oracle.mat_random_i8(case["n"], case["k"], case["seed_b"])
        assert oracle.gemm(a, b, EXACT).ravel().tolist() == case["exact"]
        assert oracle.gemm(a, b, SAT).ravel().tolist() == case["sat"]


def test_wrapping_k4096(oracle):
    # test_gemm.cpp:202-211: order independence under int32 wrap, against a numpy int64 mod 2^32
    a = oracle.mat_random_u8(2, 4096, 30)
    b = oracle.mat_random_i8(2, 4096, 31)
    ref = (a.astype(np.int64) @ b.astype(np.int64).T) & 0xFFFFFFFF
    ref = ref.astype(np.uint32).view(np.int32)
    assert (oracle.gemm(a, b, EXACT) == ref).all()


def test_pack_2x2_bytes(oracle, golden):
    # test_layout.cpp:61-84
    a = np.array([[1, 2], [3, 4]], np.uint8)
    meta = oracle.packed_meta(2, 2, w=32, h=4, v=8, tm=8, tn=1, tk=4, perm=0)
    p = oracle.pack(a, meta)
    assert p.size == 32
    assert p[:8].tolist() == [1, 2, 0, 0, 3, 4, 0, 0] and (p[8:] == 0).all()
    assert p.tolist() == golden["packs"][0]["head"][:32]


def test_pack_traversal_and_k_first(oracle):
    # test_layout.cpp:106-146
    a = np.zeros((16, 8), np.uint8)
    for r in range(16):
        for c in range(8):
            a[r, c] = (r // 8) * 2 + (c // 4) + 1
    p1 = oracle.pack(a, oracle.packed_meta(16, 8, 32, 4, 8, 8, 1, 4, 0))
    p2 = oracle.pack(a, oracle.packed_meta(16, 8, 32, 4, 8, 8, 1, 4, 5))
    assert [p1[i * 32] for i in range(4)] == [1, 2, 3, 4]
    assert [p2[i * 32] for i in range(4)] == [1, 3, 2, 4]
    p3 = oracle.pack(a, oracle.packed_meta(16, 8, 32, 4, 8, 16, 1, 8, 0))
    assert [p3[i * 32] for i in range(4)] == [1, 2, 3, 4]


def test_pack_digests_vs_reference(oracle, golden):
    for c in golden["packs"]:
        a = np.array([[1, 2], [3, 4]], np.uint8) if c["seed"] is None else oracle.mat_random_u8(c["m"], c["k"], c["seed"])
        meta = oracle.packed_meta(c["m"], c["k"], c["w"], c["h"], c["v"], c["tm"], c["tn"], c["tk"], c["perm"])
        p = oracle.pack(a, meta)
        assert p.size == c["nbytes"]
        assert oracle.fnv1a(p) == c["fnv"]
        assert (oracle.unpack(p, meta) == a).all()


def test_unpack_detects_corruption(oracle):
    # test_layout.cpp:186-193
    a = oracle.mat_random_u8(5, 5, 3, 1, 255)
    meta = oracle.packed_meta(5, 5, 32, 4, 8, 8, 1, 4, 0)
    p = oracle.pack(a, meta)
    p[oracle.elem_offset(meta, 7, 0)] = 42
    with pytest.raises(ValueError):
        oracle.unpack(p, meta)


def test_pack_config_errors(oracle):
    # test_layout.cpp:195-207
    for tm, tn, tk in ((7, 1, 4), (8, 1, 5), (8, 0, 4)):
        with pytest.raises(ValueError):
            oracle.packed_meta(4, 4, 32, 4, 8, tm, tn, tk, 0)


def test_config4_known_answers(oracle, golden):
    # SURVEY Appendix A, regenerated by the reference: every element of C is equal
    def pat(kind, rows, cols, p):
        idx = np.arange(rows * cols).reshape(rows, cols) & 1
        if kind == U8:
            return np.full((rows, cols), 255, np.uint8) if p == "all255" else np.where(idx, 255, 0).astype(np.uint8)
        if p == "all-128":
            return np.full((rows, cols), -128, np.int8)
        if p == "all127":
            return np.full((rows, cols), 127, np.int8)
        return np.where(idx, 127, -128).astype(np.int8)

    for c in golden["config4"]:
        a = pat(U8, 2, c["size"], c["a"])
        b = pat(I8, 3, c["size"], c["b"])
        assert (oracle.gemm(a, b, EXACT) == c["exact"]).all()
        assert (oracle.gemm(a, b, SAT) == c["sat"]).all()


def test_config1_digest(oracle, golden):
    a = oracle.mat_random_u8(1024, 1024, 0)
    b = oracle.mat_random_i8(1024, 1024, 1)
    ce, cs = oracle.gemm(a, b, EXACT), oracle.gemm(a, b, SAT)
    g = golden["config1"]
    assert int(ce.astype(np.int64).sum()) == g["exact_checksum"] == -37581470995
    assert int(cs.astype(np.int64).sum()) == g["sat_checksum"] == -34126294179
    assert oracle.fnv1a(ce) == g["exact_fnv"] and oracle.fnv1a(cs) == g["sat_fnv"]
    assert int((ce != cs).sum()) == g["n_differ"] == 1048565


def test_config2_normal_generator_frozen(oracle, golden):
    for c in golden["config2"]:
        b = oracle.mat_normal_i8(c["n"], c["k"], 1, 32.0)
        assert oracle.fnv1a(b) == c["b_fnv"]
    b = oracle.mat_normal_i8(768, 768, 1, 32.0).astype(np.float64)
    assert abs(b.mean()) < 0.5 and 30.0 < b.std() < 34.0


def test_config3_digests(oracle, golden):
    for c in golden["config3"][:3]:  # M=128 rows; larger ones are pinned in the GPU tests
        a = oracle.mat_random_u8(c["m"], c["k"], 0)
        b = oracle.mat_random_i8(c["n"], c["k"], 1)
        assert oracle.fnv1a(oracle.gemm(a, b, EXACT)) == c["exact_fnv"]
        assert oracle.fnv1a(oracle.gemm(a, b, SAT)) == c["sat_fnv"]


def test_oracle_matches_reference_directly(oracle):
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built (reference absent)")
    ref = Reference()
    for (m, n, k, s) in ((7, 5, 13, 1), (33, 17, 64, 2), (3, 64, 129, 3)):
        a = oracle.mat_random_u8(m, k, s)
        b = oracle.mat_random_i8(n, k, s + 100)
        assert (oracle.gemm(a, b, EXACT) == ref.gemm("gemm_ref", a, b)).all()
        assert (oracle.gemm(a, b, SAT) == ref.gemm("gemm_sat_oracle", a, b)).all()
        assert (oracle.gemm(a, b, SAT) == ref.gemm("gemm_conventional", a, b, SAT, engine=0)).all()


def test_i16_oracle_vs_reference_golden(oracle, golden):
    # inputs: the reference's mat_random(I16) restated; outputs: gemm_ref on i16 (gemm.hpp:36-52),
    # which the reference's emulated 16-bit gemm_conventional matched when the fixture was made
    for c in golden["i16"]:
        a = oracle.mat_random_i16(c["m"], c["k"], c["seed"], c["lo"], c["hi"])
        b = oracle.mat_random_i16(c["n"], c["k"], c["seed"] + 100, c["lo"], c["hi"])
        assert oracle.fnv1a(a) == c["a_fnv"]
        out = oracle.gemm_i16(a, b)
        assert oracle.fnv1a(out) == c["c_fnv"] and int(out.astype(np.int64).sum()) == c["c_sum"]

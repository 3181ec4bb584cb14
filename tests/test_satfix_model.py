"""CPU model of the saturating tensor-core decomposition (kernel_satfix.cuh).

A pair (b0, b1) of B is "dangerous" when some a0, a1 in [0, amax] can push a0*b0 + a1*b1 out
of int16.  The GPU computes C = A . B_safe (B with the dangerous pairs zeroed, exact, on the
tensor cores) + the clamped sums of the dangerous pairs (CUDA cores).  This checks, on the
CPU and against the pinned oracle (gemm_sat_oracle, gemm.hpp:83-104), that the decomposition
and the classification rule used by sat_prep_b_kernel are exact — including extremes, odd K
and inputs with amax < 255."""
import numpy as np
import pytest

from oracle.oracle import EXACT, SAT


def dangerous_pairs(b: np.ndarray, amax: int) -> np.ndarray:
    """[n, ceil(k/2)] bool, the rule of sat_prep_b_kernel: amax * pos > 32767 or amax * neg > 32768."""
    n, k = b.shape
    bp = np.zeros((n, (k + 1) // 2 * 2), np.int64)
    bp[:, :k] = b
    b0, b1 = bp[:, 0::2], bp[:, 1::2]
    pos = np.maximum(b0, 0) + np.maximum(b1, 0)
    neg = -(np.minimum(b0, 0) + np.minimum(b1, 0))
    return (amax * pos > 32767) | (amax * neg > 32768)


def hybrid_model(a: np.ndarray, b: np.ndarray, oracle) -> np.ndarray:
    m, k = a.shape
    d = dangerous_pairs(b, int(a.max()) if a.size else 0)
    dk = np.repeat(d, 2, axis=1)[:, :k]  # per element of B
    b_safe = np.where(dk, 0, b).astype(np.int8)
    c = oracle.gemm(a, b_safe, EXACT).astype(np.int64)  # the tensor-core term
    # the fix term: clamped pair sums of the dangerous pairs only
    kp = (k + 1) // 2 * 2
    ap = np.zeros((m, kp), np.int64)
    ap[:, :k] = a
    bp = np.zeros((b.shape[0], kp), np.int64)
    bp[:, :k] = b
    pair = ap[:, None, 0::2] * bp[None, :, 0::2] + ap[:, None, 1::2] * bp[None, :, 1::2]  # [m, n, k/2]
    fix = np.where(d[None, :, :], np.clip(pair, -32768, 32767), 0).sum(axis=2)
    return ((c + fix + 2**31) % 2**32 - 2**31).astype(np.int32)


@pytest.mark.parametrize("case", ["uniform", "normal", "extreme", "small_amax", "odd_k"])
def test_decomposition_matches_sat_oracle(oracle, case):
    rng = np.random.default_rng(7)
    m, n, k = 37, 29, 258
    a = rng.integers(0, 256, (m, k), dtype=np.uint8)
    if case == "uniform":
        b = rng.integers(-128, 128, (n, k), dtype=np.int8)
    elif case == "normal":
        b = np.clip(np.rint(rng.normal(0, 32, (n, k))), -128, 127).astype(np.int8)
    elif case == "extreme":
        a[:] = 255
        b = np.where(rng.random((n, k)) < 0.5, 127, -128).astype(np.int8)
    elif case == "small_amax":  # amax = 129: only |b0 + b1|-heavy pairs are dangerous
        a = rng.integers(0, 130, (m, k), dtype=np.uint8)
        b = rng.integers(-128, 128, (n, k), dtype=np.int8)
    else:
        k = 257
        a = rng.integers(0, 256, (m, k), dtype=np.uint8)
        b = rng.integers(-128, 128, (n, k), dtype=np.int8)
    assert (hybrid_model(a, b, oracle) == oracle.gemm(a, b, SAT)).all()


def test_classification_is_tight_at_the_int16_edges():
    """Pairs exactly at the edge stay safe; one step past it is dangerous (amax = 255: pos <= 128)."""
    b = np.array([[64, 64, 65, 64, -64, -64, -65, -64, 127, 1, -128, 0, -128, -1]], np.int8)
    d = dangerous_pairs(b, 255)[0].tolist()
    # 255*128 = 32640 ok; 255*129 = 32895 > 32767; neg 128 ok (32640 <= 32768); 129 not
    assert d == [False, True, False, True, False, False, True]
    # amax 0: nothing can clamp
    assert not dangerous_pairs(b, 0).any()

"""One-off soak of tests/test_gpu_parity.py::test_dispatcher_fuzz_auto's generator with other seeds
(run on a B200): python scripts/fuzz_soak.py [first_seed] [seeds]"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle.oracle import EXACT, SAT, Oracle
import test_gpu_parity as T

def main():
    first = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    ora = Oracle()
    total = 0
    t0 = time.time()
    for seed in range(first, first + count):
        rng = np.random.default_rng(seed)
        pick = lambda lo, hi: int(np.exp(rng.uniform(np.log(lo), np.log(hi))))
        for it in range(160):
            kind = it % 4
            if kind == 0:
                m, n, k = int(rng.integers(1, 17)), pick(1, 6000), pick(1, 20000)
            elif kind == 1:
                m, n, k = pick(17, 700), pick(1, 1500), pick(1, 3000)
            elif kind == 2:
                m, n, k = pick(17, 300), pick(500, 5000), pick(500, 9000)
            else:
                m, n, k = pick(200, 1200), pick(700, 1500), pick(700, 1500)
            while 2.0 * m * n * k > 6e9:
                k = max(1, k // 2)
            pad = int(rng.integers(0, 3))
            lda = k + (0 if pad == 0 else int(rng.integers(1, 40)))
            ldb = k + (0 if pad == 0 else int(rng.integers(1, 40)))
            ldc = n + (0 if pad != 2 else int(rng.integers(1, 9)))
            a = ora.mat_random_u8(m, k, seed * 100000 + it)
            b = ora.mat_normal_i8(n, k, seed * 100000 + 50000 + it, 32.0) if it % 3 else ora.mat_random_i8(n, k, seed * 100000 + 50000 + it)
            for mode in (EXACT, SAT):
                got = T.dev_gemm(a, b, mode, "auto", lda, ldb, ldc)
                if not (got == ora.gemm(a, b, mode)).all():
                    print("MISMATCH", seed, it, m, n, k, lda, ldb, ldc, mode, flush=True)
                    sys.exit(1)
                total += 1
        print(f"seed {seed}: ok ({total} GEMMs so far, {time.time() - t0:.0f} s)", flush=True)
    print(f"fuzz soak: {total} GEMMs bit-exact vs the oracle")

main()

"""Canary probe: which kernels write past column N-1 when ldc > N (the TMA-epilogue granule issue)."""
import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, ".")
import numpy as np
sys.path.insert(0, "tests")
from test_gpu_parity import dev_gemm
from oracle.oracle import Oracle, EXACT, SAT
from paper_1910_00178_b200 import _lib  # noqa: E402
ora = Oracle()
rng = np.random.default_rng(0)
for (m, n, k) in [(300, 333, 777), (512, 640, 1024), (256, 200, 512)]:
    a = rng.integers(0, 256, (m, k), dtype=np.uint8)
    b = rng.integers(-128, 128, (n, k), dtype=np.int8)
    for kern, mode, env in [("tcgen05", EXACT, "-1"), ("sat_hybrid", SAT, "-1"), ("simt", SAT, "-1")]:
        for ldc in (n + 3, n + 7, n + 19):
            if ldc % 4: continue
            _lib.set_option("SAT_HYBRID", int(env))
            try:
                got = dev_gemm(a, b, mode, kern, ldc=ldc)
                ok = (got == ora.gemm(a, b, mode)).all()
                print(m, n, k, kern, ldc, "ok" if ok else "MISMATCH")
            except AssertionError as e:
                print(m, n, k, kern, ldc, "CANARY", e)
            except Exception as e:  # sat_hybrid refuses N % 4 != 0
                print(m, n, k, kern, ldc, "refused:", type(e).__name__)
    for skip in ("1", "2", "8", "16"):
        _lib.set_option("SATFIX_SKIP", int(skip))
        try:
            dev_gemm(a, b, SAT, "sat_hybrid", ldc=n + 3)
            print("skip", skip, "no canary hit")
        except AssertionError as e:
            print("skip", skip, "CANARY", str(e)[:60])
        except Exception as e:
            print("skip", skip, "refused:", type(e).__name__)
    _lib.reset_options()

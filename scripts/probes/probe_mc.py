"""1-CTA A-multicast cluster configs (NGEMM_TC_CFG=7: 128x128, 8: 128x64): bit-exact check on a
few shapes, then kernel times against the planner's default on c1/c3 shapes (CUDA graph)."""
import os
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np  # noqa: E402

from oracle.oracle import EXACT, Oracle  # noqa: E402
from paper_1910_00178_b200 import _lib  # noqa: E402
from test_gpu_parity import dev_gemm  # noqa: E402

ora = Oracle()
for cfg in ("7", "8"):
    _lib.set_option("TC_CFG", int(cfg))
    for (m, n, k) in ((256, 256, 256), (300, 512, 1100), (1024, 1024, 1024), (129, 640, 640)):
        a = ora.mat_random_u8(m, k, 3)
        b = ora.mat_random_i8(n, k, 4)
        got = dev_gemm(a, b, EXACT, "tcgen05")
        print("cfg", cfg, m, n, k, "ok" if (got == ora.gemm(a, b, EXACT)).all() else "MISMATCH", flush=True)
_lib.reset_options()

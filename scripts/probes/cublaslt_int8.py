"""Library reference point (not the product): cuBLASLt int8 GEMM through torch._int_mm
(s8 x s8 -> s32; cuBLASLt has no u8 x s8 kind) on the config-5 and config-3 shapes, timed
with CUDA events after warm-up, next to this repo's tcgen05 kernel on the same shapes."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_00178_b200 import api  # noqa: E402


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


import time

for (m, n, k, reps) in [(4096, 4096, 4096, 200), (8192, 8192, 8192, 50), (12288, 12288, 12288, 20),
                        (16384, 16384, 16384, 20), (8192, 8192, 8192, 50)]:
    a8 = torch.randint(-128, 128, (m, k), dtype=torch.int8, device="cuda")
    bt = torch.randint(-128, 128, (k, n), dtype=torch.int8, device="cuda")  # _int_mm wants [k, n]
    au = torch.randint(0, 256, (m, k), dtype=torch.int32, device="cuda").to(torch.uint8)
    b = torch.randint(-128, 128, (n, k), dtype=torch.int8, device="cuda")
    c = torch.empty((m, n), dtype=torch.int32, device="cuda")
    ops = 2.0 * m * n * k
    row = {"shape": f"{m}x{n}x{k}"}
    for name, fn in (("ours_tcgen05_tops", lambda: api.gemm_device(au, b, c)),
                     ("cublaslt_int_mm_tops", lambda: torch._int_mm(a8, bt)),
                     ("ours_tcgen05_tops_again", lambda: api.gemm_device(au, b, c))):
        time.sleep(0.5)  # let the clocks recover between arms
        row[name] = round(ops / timeit(fn, reps) / 1e12, 1)
    print(json.dumps(row), flush=True)

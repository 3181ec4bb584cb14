"""Fused requantisation epilogue vs the int32 GEMM (and vs GEMM + a separate requant pass), same
shapes, CUDA-graph timed over a rotating pool of operand sets (> 4x L2)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_00178_b200 import api  # noqa: E402
from paper_1910_00178_b200 import _lib  # noqa: E402


def timed(fn, reps, graph=True):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(3):
            fn(i)
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(reps):
                fn(i)
        g.replay()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if graph:
        g.replay()
    else:
        for i in range(reps):
            fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


dev = torch.device("cuda")
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
for (m, n, k) in [(2048, 4096, 1024), (2048, 1024, 4096), (512, 4096, 1024), (1024, 1024, 1024), (8192, 8192, 8192),
                  (16, 4096, 1024), (4, 3072, 768), (1, 4096, 1024)]:
    per = m * k + n * k + 4 * m * n
    nb = 1 if per > 2 * l2 else min(16, int(4 * l2 // per) + 1)
    A = [torch.randint(0, 256, (m, k), dtype=torch.int32, device=dev).to(torch.uint8) for _ in range(nb)]
    B = [torch.randint(-128, 128, (n, k), dtype=torch.int32, device=dev).to(torch.int8) for _ in range(nb)]
    C = [torch.empty((m, n), dtype=torch.int32, device=dev) for _ in range(nb)]
    O = [torch.empty((m, n), dtype=torch.int8, device=dev) for _ in range(nb)]
    sc = torch.full((n,), 1.0 / 2000.0, dtype=torch.float32, device=dev)
    bi = torch.zeros(n, dtype=torch.int32, device=dev)
    reps = 20 if m * n * k < 2**33 else 5
    big = m * n * k >= 2**33
    t_gemm = timed(lambda i: api.gemm_device(A[i % nb], B[i % nb], C[i % nb]), reps, not big)
    t_rq = timed(lambda i: api.gemm_device_requant(A[i % nb], B[i % nb], sc, bi, 0, out=O[i % nb]), reps, not big)
    _lib.set_option("REQUANT_UNFUSED", 1)  # int32 C in scratch, then requant_kernel
    t_un = timed(lambda i: api.gemm_device_requant(A[i % nb], B[i % nb], sc, bi, 0, out=O[i % nb]), reps, not big)
    _lib.reset_options()
    print(json.dumps({"shape": f"{m}x{n}x{k}", "int32_gemm_us": round(t_gemm, 2), "fused_requant_us": round(t_rq, 2),
                      "unfused_requant_us": round(t_un, 2),
                      "out_bytes_int32": 4 * m * n, "out_bytes_int8": m * n}), flush=True)

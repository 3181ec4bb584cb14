"""Library reference point (not the product): cuBLASLt int8 (torch._int_mm, s8 x s8 -> s32) vs
this repo's kernels on the medium / compute shapes, both CUDA-graph timed over rotating buffer
sets > 4x L2 (every launch L2-cold), same box, interleaved."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_00178_b200 import api  # noqa: E402

L2 = torch.cuda.get_device_properties(0).L2_cache_size


def graph_time(launch, nbuf, reps):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(3):
            launch(i % nbuf)
        with torch.cuda.graph(g, stream=s):
            for i in range(reps):
                launch(i % nbuf)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


shapes = sys.argv[1:] or ["1024x1024x1024", "2048x2048x2048", "4096x4096x4096", "128x1024x1024", "128x4096x1024",
                          "128x1024x4096", "512x1024x1024", "512x4096x1024", "512x1024x4096", "2048x1024x1024",
                          "2048x4096x1024", "2048x1024x4096", "8192x8192x8192"]
for sh in shapes:
    m, n, k = (int(x) for x in sh.split("x"))
    per = m * k + n * k + 4 * m * n
    nbuf = max(1, min(256, int(4 * L2 // per) + 1))
    reps = max(20, nbuf) if per < 2 * L2 else 10
    au = [torch.randint(0, 256, (m, k), dtype=torch.int32, device="cuda").to(torch.uint8) for _ in range(nbuf)]
    b = [torch.randint(-128, 128, (n, k), dtype=torch.int8, device="cuda") for _ in range(nbuf)]
    c = [torch.empty((m, n), dtype=torch.int32, device="cuda") for _ in range(nbuf)]
    a8 = [x.view(torch.int8) for x in au]
    bt = [x.t() for x in b]  # _int_mm wants [k, n]; a transposed view is the column-major operand
    ops = 2.0 * m * n * k
    row = {"shape": sh}
    for rep in range(2):
        t_ours = graph_time(lambda i: api.gemm_device(au[i], b[i], c[i]), nbuf, reps)
        t_lt = graph_time(lambda i: torch._int_mm(a8[i], bt[i]), nbuf, reps)
        row[f"ours_us_{rep}"] = round(t_ours, 2)
        row[f"cublaslt_us_{rep}"] = round(t_lt, 2)
    row["ours_tops"] = round(ops / (min(row["ours_us_0"], row["ours_us_1"]) * 1e-6) / 1e12, 1)
    row["cublaslt_tops"] = round(ops / (min(row["cublaslt_us_0"], row["cublaslt_us_1"]) * 1e-6) / 1e12, 1)
    row["ratio"] = round(row["ours_tops"] / row["cublaslt_tops"], 3)
    print(json.dumps(row), flush=True)

"""Throughput of the strided-batched skinny GEMM (ngemm_cuda_gemm_u8i8_strided_batched) versus
the same GEMMs issued one launch at a time.

For each (M, N, K) and batch size G the whole batch's operands exceed L2 (126 MB) once
G * N * K > 256 MB, so every timed launch streams B from HBM; smaller G rotate over 4 copies
of the batch so successive launches do not hit in L2.  Prints one line per point:
  shape G  us_per_batch  GB/s(algorithmic: G*(N*K + M*K + 4*M*N))  frac_of_hbm  us_looped
Run on a B200:  python scripts/batched_probe.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_00178_b200 import _lib  # noqa: E402

L2_BYTES = 126 << 20


def hbm_peak():
    try:
        d = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
        for key in ("hbm_gbs",):
            if key in d:
                return float(d[key])
    except Exception:
        pass
    return 6650.0  # B200_PROFILING.md fallback


def main():
    L = _lib.load()
    peak = hbm_peak()
    shapes = [(1, 4096, 4096), (8, 4096, 1024), (16, 4096, 1024), (16, 8192, 4096), (4, 1024, 4096)]
    modes = [int(x) for x in os.environ.get("PROBE_MODES", "1,0").split(",")]
    for mode in modes:
        for (m, n, k) in shapes:
            for g in [int(x) for x in os.environ.get("PROBE_G", "1,8,32,128").split(",")]:
                per = n * k + m * k + 4 * m * n
                copies = max(1, min(4, (2 * L2_BYTES) // max(1, g * per) + 1))
                a = torch.randint(0, 256, (copies, g, m, k), dtype=torch.uint8, device="cuda")
                b = torch.randint(-128, 128, (copies, g, n, k), dtype=torch.int8, device="cuda")
                c = torch.empty((copies, g, m, n), dtype=torch.int32, device="cuda")

                def batched(i):
                    _lib.check(L.ngemm_cuda_gemm_u8i8_strided_batched(
                        a[i].data_ptr(), k, m * k, b[i].data_ptr(), k, n * k, c[i].data_ptr(), n, m * n, g, m, n,
                        k, mode, torch.cuda.current_stream().cuda_stream))

                def looped(i):
                    for z in range(g):
                        _lib.check(L.ngemm_cuda_gemm_u8i8(a[i, z].data_ptr(), k, b[i, z].data_ptr(), k,
                                                          c[i, z].data_ptr(), n, m, n, k, mode, torch.cuda.current_stream().cuda_stream))

                res = []
                for fn in (batched, looped):
                    for i in range(3):
                        fn(i % copies)
                    graph = torch.cuda.CUDAGraph()
                    reps = 20
                    with torch.cuda.graph(graph):
                        for r in range(reps):
                            fn(r % copies)
                    graph.replay()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(5):
                        graph.replay()
                    e1.record()
                    torch.cuda.synchronize()
                    res.append(e0.elapsed_time(e1) * 1e3 / (5 * reps))
                us, us_loop = res
                gbps = g * per / (us * 1e-6) / 1e9
                print(f"mode={'exact' if mode else 'sat'} {m}x{n}x{k} G={g:4d} batched {us:9.2f} us "
                      f"{gbps:8.1f} GB/s frac {gbps / peak:.3f}  looped {us_loop:9.2f} us", flush=True)
                del a, b, c
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

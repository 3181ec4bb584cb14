"""i16 x i16 GEMM throughput: CUDA-core kernel vs the tensor-core byte-plane decomposition.
Run on a B200: python scripts/i16_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_00178_b200 import _lib  # noqa: E402


def main():
    L = _lib.load()
    for (m, n, k) in [(1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096), (8192, 8192, 8192)]:
        a = torch.randint(-32768, 32768, (m, k), dtype=torch.int16, device="cuda")
        b = torch.randint(-32768, 32768, (n, k), dtype=torch.int16, device="cuda")
        c = torch.empty((m, n), dtype=torch.int32, device="cuda")
        res = {}
        for path in ("simt", "tcgen05"):
            if path == "simt" and m * n * k > 4096 ** 3:
                continue
            _lib.set_option("I16_PATH", {"tcgen05": 1, "simt": 0}.get(path, path))

            def run():
                _lib.check(L.ngemm_cuda_gemm_i16(a.data_ptr(), k, b.data_ptr(), k, c.data_ptr(), n, m, n, k,
                                                 torch.cuda.current_stream().cuda_stream))
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            reps = 10
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / reps
            res[path] = us
            print(f"i16 {m}x{n}x{k} {path:8s} {us:10.1f} us  {2 * m * n * k / us / 1e6:8.1f} TOPS", flush=True)
        if len(res) == 2:
            print(f"   speed-up {res['simt'] / res['tcgen05']:.1f}x")


if __name__ == "__main__":
    main()

"""Phase trace of the tcgen05 GEMM kernel inside a CUDA graph of back-to-back launches.

Loads the trace build of the library (`make trace` -> libngemm_cuda_trace.so: the production
kernel with %globaltimer stamps compiled in) and prints, per shape, where a launch's time goes
(all times in us relative to the launch's first CTA entry, averaged over steady-state launches):
  setup   = barrier init + TMEM alloc + cluster sync done
  release = PDL wait returns
  data    = first operand stage lands at the MMA issuer
  mma     = last MMA committed
  epi     = first accumulator ready / last TMA store drained
  exit    = CTA exit;  gap = last exit of launch L -> first release of launch L+1
Run on a B200:  make trace && python scripts/probes/tc_trace.py [MxNxK ...]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
L_MAX, CTA_MAX, NP = 64, 160, 16


def main():
    lib = C.CDLL(os.path.join(ROOT, "paper_1910_00178_b200", "lib", "libngemm_cuda_trace.so"))
    vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
    lib.ngemm_cuda_gemm_u8i8_ex.argtypes = [vp, i64, vp, i64, vp, i64, i64, i64, i64, i32, i32, vp]
    lib.ngemm_trace_read.argtypes = [vp, C.c_size_t]
    shapes = sys.argv[1:] or ["128x1024x1024", "512x4096x1024", "2048x4096x1024", "2048x2048x2048",
                              "1024x1024x1024", "16384x16384x16384"]
    for sh in shapes:
        m, n, k = (int(x) for x in sh.split("x"))
        per = m * k + n * k + 4 * m * n
        nb = max(1, min(8, (512 << 20) // per))
        R = 48 if per < (1 << 30) else 12
        a = [torch.randint(0, 256, (m, k), dtype=torch.uint8, device="cuda") for _ in range(nb)]
        b = [torch.randint(-128, 128, (n, k), dtype=torch.int8, device="cuda") for _ in range(nb)]
        c = [torch.empty((m, n), dtype=torch.int32, device="cuda") for _ in range(nb)]

        def launch(i):
            rc = lib.ngemm_cuda_gemm_u8i8_ex(a[i % nb].data_ptr(), k, b[i % nb].data_ptr(), k, c[i % nb].data_ptr(),
                                             n, m, n, k, 1, 1, torch.cuda.current_stream().cuda_stream)
            assert rc == 0, rc

        for i in range(3):
            launch(i)
        assert lib.ngemm_trace_reset() == 0  # captured launches get trace ids 0..R-1
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(R):
                launch(i)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / R
        buf = np.zeros((L_MAX, CTA_MAX, NP), dtype=np.uint64)
        assert lib.ngemm_trace_read(buf.ctypes.data, buf.nbytes) == 0
        t = buf.astype(np.float64)
        t[t == 0] = np.nan
        rows = []
        for L in range(2, min(R, L_MAX) - 2):
            t0 = np.nanmin(t[L, :, 0])
            mn = lambda p: np.nanmin(t[L, :, p]) - t0  # noqa: E731
            mx = lambda p: np.nanmax(t[L, :, p]) - t0  # noqa: E731
            gap = np.nanmin(t[L + 1, :, 2]) - np.nanmax(t[L, :, 9])
            rows.append([mx(0), mx(1), mn(2), mx(2), mn(5), mx(5), mx(6), mn(7), mx(8), mx(9), gap,
                         mn(10), mn(11), mn(12)])
        r = np.nanmean(np.array(rows), axis=0) / 1e3
        ctas = int(np.sum(~np.isnan(t[4, :, 0])))
        print(f"{sh:>18s} {us:8.2f} us/launch ({ctas} CTAs) | entry<= {r[0]:.2f} setup<= {r[1]:.2f} "
              f"release {r[2]:.2f}..{r[3]:.2f} data {r[4]:.2f}..{r[5]:.2f} mma-done {r[6]:.2f} "
              f"epi-first {r[7]:.2f} epi-done {r[8]:.2f} exit {r[9]:.2f} | gap {r[10]:.2f} | first tile, warp 4: "
              f"tmem-ld {r[11]:.2f} store0 {r[12]:.2f} tile-stores-issued {r[13]:.2f}", flush=True)
        del a, b, c, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

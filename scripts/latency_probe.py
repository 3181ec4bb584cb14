"""Where does the time of a skinny GEMM go?  eager vs graph, PDL on/off, 1 vs 4 streams."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1910_00178_b200 import api, _lib
m, n, k = (int(x) for x in sys.argv[1].split("x"))
kern = int(sys.argv[2]) if len(sys.argv) > 2 else 0
R = 200
dev = torch.device("cuda")
nbuf = 64
A = [torch.randint(0, 256, (m, k), device=dev, dtype=torch.int32).to(torch.uint8) for _ in range(nbuf)]
B = [torch.randint(-128, 128, (n, k), device=dev, dtype=torch.int32).to(torch.int8) for _ in range(nbuf)]
C = [torch.empty((m, n), device=dev, dtype=torch.int32) for _ in range(nbuf)]
s0 = torch.cuda.current_stream()
def run(i, st):
    api.gemm_device(A[i % nbuf], B[i % nbuf], C[i % nbuf], mode=1, kernel=kern, stream=st)
for i in range(20): run(i, s0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); [run(i, s0) for i in range(R)]; e1.record(); torch.cuda.synchronize()
print(f"eager   1 stream : {e0.elapsed_time(e1) * 1000 / R:7.2f} us/gemm")
g = torch.cuda.CUDAGraph(); cap = torch.cuda.Stream()
with torch.cuda.stream(cap):
    with torch.cuda.graph(g, stream=cap):
        for i in range(R): run(i, cap)
g.replay(); torch.cuda.synchronize()
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
print(f"graph   1 stream : {e0.elapsed_time(e1) * 1000 / R:7.2f} us/gemm")
streams = [torch.cuda.Stream() for _ in range(4)]
g2 = torch.cuda.CUDAGraph()
with torch.cuda.stream(cap):
    with torch.cuda.graph(g2, stream=cap):
        for st in streams: st.wait_stream(cap)
        for i in range(R):
            run(i, streams[i % 4])
        for st in streams: cap.wait_stream(st)
g2.replay(); torch.cuda.synchronize()
e0.record(); g2.replay(); e1.record(); torch.cuda.synchronize()
print(f"graph   4 streams: {e0.elapsed_time(e1) * 1000 / R:7.2f} us/gemm  (bytes/gemm {n*k + m*k + 4*m*n})")

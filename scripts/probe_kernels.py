"""Runs one kernel family on one small shape and compares with the oracle (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.oracle import Oracle
from paper_1910_00178_b200 import _lib, api
kern = {"simt": 2, "tcgen05": 1, "skinny": 3, "auto": 0}[sys.argv[1]]
m, n, k = (int(x) for x in sys.argv[2].split("x"))
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 1
o = Oracle()
a = o.mat_random_u8(m, k, 0); b = o.mat_random_i8(n, k, 1)
c = api.gemm_device(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), mode=mode, kernel=kern)
torch.cuda.synchronize()
ref = o.gemm(a, b, mode); got = c.cpu().numpy()
bad = int((got != ref).sum())
print(f"{sys.argv[1]} {m}x{n}x{k} mode={mode}: {'OK' if bad == 0 else 'MISMATCH %d' % bad}")
if bad:
    idx = np.argwhere(got != ref)[:5]
    for i, j in idx: print("  ", i, j, got[i, j], ref[i, j])

"""Small invocations of every kernel family for compute-sanitizer (one tool per gpurun call)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.oracle import Oracle
from paper_1910_00178_b200 import _lib, api
o = Oracle()
cases = [(300, 520, 1100, 1, 1), (256, 256, 2048, 1, 1), (129, 65, 640, 0, 2), (16, 300, 777, 1, 3), (5, 300, 777, 0, 3),
         (300, 300, 300, 0, 0)]
for (m, n, k, mode, kern) in cases:
    a = o.mat_random_u8(m, k, 1); b = o.mat_random_i8(n, k, 2)
    c = api.gemm_device(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), mode=mode, kernel=kern)
    torch.cuda.synchronize()
    assert (c.cpu().numpy() == o.gemm(a, b, mode)).all(), (m, n, k, mode, kern)
for v in ("0", "1", "2", "3", "4"):
    _lib.set_option("SKINNY_VARIANT", int(v))
    for mode in (0, 1):
        a = o.mat_random_u8(7, 1000, 3); b = o.mat_random_i8(200, 1000, 4)
        c = api.gemm_device(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), mode=mode, kernel=3)
        torch.cuda.synchronize()
        assert (c.cpu().numpy() == o.gemm(a, b, mode)).all(), (v, mode)
_lib.reset_options()
_lib.set_option("TC_CFG", 0)
a = o.mat_random_u8(512, 256, 5); b = o.mat_random_i8(512, 256, 6)
c = api.gemm_device(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), mode=1, kernel=1)
torch.cuda.synchronize()
assert (c.cpu().numpy() == o.gemm(a, b, 1)).all()
print("sanitize probe: all kernels bit-exact")

"""A few fused-requant GEMMs (2048x4096x1024) for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1910_00178_b200 import api  # noqa: E402

m, n, k = 2048, 4096, 1024
a = torch.randint(0, 256, (m, k), dtype=torch.int32, device="cuda").to(torch.uint8)
b = torch.randint(-128, 128, (n, k), dtype=torch.int32, device="cuda").to(torch.int8)
sc = torch.full((n,), 1.0 / 2000.0, dtype=torch.float32, device="cuda")
for _ in range(3):
    api.gemm_device_requant(a, b, sc)
torch.cuda.synchronize()
print("ok")

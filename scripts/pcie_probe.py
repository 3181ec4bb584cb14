"""PCIe probe: pinned H2D / D2H bandwidth alone and concurrently (the e2e bound of bench.py)."""
import torch


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


h_in = torch.empty(512 << 20, dtype=torch.uint8).pin_memory()
h_out = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
d_in = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
d_out = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ms = t(lambda: d_in.copy_(h_in, non_blocking=True))
print(f"H2D 512 MiB: {ms:.2f} ms  {512 / 1024 / ms * 1e3:.1f} GiB/s")
ms = t(lambda: h_out.copy_(d_out, non_blocking=True))
print(f"D2H 1 GiB:   {ms:.2f} ms  {1 / ms * 1e3:.1f} GiB/s")


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


ms = t(both)
print(f"H2D 512 MiB || D2H 1 GiB: {ms:.2f} ms")

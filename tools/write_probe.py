"""Write-only and read-only HBM ceilings on this B200 (tooling): the roofline of
the launch-control sweep (16 B written per amplitude, nothing read) is the
write bandwidth, not the copy bandwidth.  16 GiB buffer (N=30 state), CUDA
events, best of 10."""
import torch

nbytes = 16 << 30
a = torch.empty(nbytes // 16, dtype=torch.complex128, device="cuda")
b = torch.empty(nbytes // 2 // 16, dtype=torch.complex128, device="cuda")


def t(fn, reps=10):
    best = 1e9
    for _ in range(reps + 2):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


ms = t(lambda: a.fill_(0.5 + 0.25j))
print(f"fill_ (write only) 16 GiB: {ms:.3f} ms = {nbytes / ms / 1e6:.0f} GB/s")
ms = t(lambda: a.zero_())
print(f"zero_ (memset) 16 GiB: {ms:.3f} ms = {nbytes / ms / 1e6:.0f} GB/s")
ms = t(lambda: torch.sum(a.view(torch.float64)))
print(f"sum (read only) 16 GiB: {ms:.3f} ms = {nbytes / ms / 1e6:.0f} GB/s")
h = a[: nbytes // 2 // 16]
ms = t(lambda: b.copy_(h))
print(f"copy 8 GiB -> 8 GiB (read+write 16 GiB): {ms:.3f} ms = {nbytes / ms / 1e6:.0f} GB/s")

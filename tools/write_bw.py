"""Diagnostic: device write-only and read-only bandwidth (torch fill_ / sum over
8 GiB, CUDA events) -- the ceilings for the apply pass and the scan."""
import torch
x = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in [("fill_ (write)", lambda: x.fill_(0)), ("view int64 sum (read)", lambda: x.view(torch.int64).sum())]:
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {best:.3f} ms  {x.numel() / best / 1e6:.0f} GB/s")

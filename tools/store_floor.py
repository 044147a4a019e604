#!/usr/bin/env python3
"""Write-bandwidth floor for the bench's output (80 MB f64) after the same
256 MiB L2 flush the bench uses: torch fill_ and a copy, CUDA events."""
import torch

n = 10_000_000
out = torch.empty(n, dtype=torch.float64, device="cuda")
src = torch.empty(n, dtype=torch.float64, device="cuda").fill_(2.0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for name, fn in (("fill", lambda: out.fill_(1.0)), ("copy", lambda: out.copy_(src)),
                 ("fill_noflush", lambda: out.fill_(3.0))):
    ts = []
    for i in range(12):
        if name != "fill_noflush":
            flush.zero_()
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(ev[0].elapsed_time(ev[1]))
    t = sorted(ts)[len(ts) // 2]
    print(f"{name}: {t*1e3:.1f} us  -> {8*n/t/1e6:.0f} GB/s (written bytes)")

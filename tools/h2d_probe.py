"""Measurement tool: pinned host -> device copy bandwidth (the e2e bound)."""
import torch, time
dev = torch.device("cuda", 0)
for mb in (64, 256, 1024):
    h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); n = 10
    for _ in range(n): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(f"H2D {mb} MiB: {n * (mb << 20) / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
    for _ in range(3): h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n): h.copy_(d, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print(f"D2H {mb} MiB: {n * (mb << 20) / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")

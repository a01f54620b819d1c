"""Pinned host->device copy bandwidth for the bench's per-step input size
(the e2e bound when compute overlaps the copies)."""
import torch
n = 12_595_712
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    d.copy_(h, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"H2D {n/1e6:.1f} MB: {ms:.3f} ms per copy, {n/ms/1e6:.1f} GB/s")

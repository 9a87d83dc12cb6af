"""D2H copy bandwidth into pinned host memory (the e2e leg of bench.py)."""
import torch
x = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # 256 MiB
h = torch.empty(x.numel(), dtype=torch.uint8, pin_memory=True)
for _ in range(3):
    h.copy_(x, non_blocking=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    h.copy_(x, non_blocking=True)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
print(f"D2H pinned: {x.numel() / ms / 1e6:.1f} GB/s")

"""Device copy of the config-2 signal (2^26 f32 in, 2^26 out) for context: python scripts/copy_probe.py"""
import torch

x = torch.empty(1 << 26, dtype=torch.float32, device="cuda").uniform_()
y = torch.empty_like(x)
for _ in range(3):
    y.copy_(x)
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        y.copy_(x)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / 10)
ms = sorted(ts)[2]
print(f"copy 2^26 f32: {ms:.4f} ms, {2 * 4 * (1 << 26) / ms / 1e6:.0f} GB/s (read + write)")

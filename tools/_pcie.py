"""Raw pinned host -> device copy bandwidth (one and two concurrent streams), for the e2e bound."""
import torch

for mb in (4, 16, 64):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    b.record()
    b.synchronize()
    print(f"H2D {mb:3d} MB: {10 * n / (a.elapsed_time(b) / 1e3) / 1e9:.1f} GB/s")
    s2 = torch.cuda.Stream()
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    a.record()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            d2.copy_(h2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
    b.record()
    b.synchronize()
    print(f"H2D {mb:3d} MB x2 streams: {20 * n / (a.elapsed_time(b) / 1e3) / 1e9:.1f} GB/s")

"""Raw host→device copy bandwidth from pinned memory (the e2e ceiling): 2 GiB in chunks of 16–256 MiB on one
stream and on two streams. usage: python tools/h2d_probe.py (on the GPU box)"""
import torch, time
n = 1 << 31
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for chunk in (1 << 24, 1 << 26, 1 << 27, 1 << 28):
    torch.cuda.synchronize()
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for o in range(0, n, chunk):
            d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
        e1.record(); torch.cuda.synchronize()
    print("H2D chunk", chunk, "GB/s", round(n / e0.elapsed_time(e1) / 1e6, 2))
s2 = torch.cuda.Stream()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
half = n // 2
with torch.cuda.stream(s2):
    for o in range(half, n, 1 << 26):
        d[o:o + (1 << 26)].copy_(h[o:o + (1 << 26)], non_blocking=True)
for o in range(0, half, 1 << 26):
    d[o:o + (1 << 26)].copy_(h[o:o + (1 << 26)], non_blocking=True)
torch.cuda.current_stream().wait_stream(s2)
e1.record(); torch.cuda.synchronize()
print("H2D two streams GB/s", round(n / e0.elapsed_time(e1) / 1e6, 2))

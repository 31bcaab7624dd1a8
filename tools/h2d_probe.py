"""Pinned host->device copy bandwidth on the box (1.2 GB, 1-3 streams, 16-200 MB chunks): the e2e ceiling."""
import torch, time
n = 1200 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def run(k, chunk=200 << 20):
    torch.cuda.synchronize()
    t = time.perf_counter()
    streams = [s1, s2, s3][:k]
    for i, o in enumerate(range(0, n, chunk)):
        with torch.cuda.stream(streams[i % k]):
            d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
    torch.cuda.synchronize()
    return n / (time.perf_counter() - t) / 1e9
for k in (1, 2, 3):
    for chunk in (16 << 20, 64 << 20, 200 << 20):
        r = [run(k, chunk) for _ in range(5)]
        print(k, chunk >> 20, "MB", round(max(r), 1), round(sorted(r)[2], 1), "GB/s")

"""Pinned host -> device copy bandwidth, one stream vs several (the e2e ceiling)."""
import torch, time
n = 819200000 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for trial in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    one = time.perf_counter() - t
    for k in (2, 4, 8):
        torch.cuda.synchronize(); t = time.perf_counter()
        ch = (n + k - 1) // k
        streams = [torch.cuda.Stream() for _ in range(k)]
        for i in range(k):
            with torch.cuda.stream(streams[i]):
                d[i*ch:(i+1)*ch].copy_(h[i*ch:(i+1)*ch], non_blocking=True)
        torch.cuda.synchronize()
        multi = time.perf_counter() - t
        print(f"1 stream {819.2/one/1e3:.1f} GB/s, {k} streams {819.2/multi/1e3:.1f} GB/s")

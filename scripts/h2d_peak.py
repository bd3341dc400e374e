"""Pinned host <-> device copy bandwidth on this box (the e2e bound): 1.6 GB H2D, 200 MB D2H,
and both at once on two streams."""
import torch, time, json
n = 1_600_000_000
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
hp = torch.empty(200_000_000, dtype=torch.uint8, pin_memory=True)
dp = torch.empty(200_000_000, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, k=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k
h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: hp.copy_(dp, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): hp.copy_(dp, non_blocking=True)
bt = t(both)
print(json.dumps({"h2d_GBs": n / h2d / 1e9, "d2h_GBs": 2e8 / d2h / 1e9, "h2d_ms": h2d * 1e3, "both_ms": bt * 1e3}))

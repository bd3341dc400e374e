"""Per-pass cost of the LSD sort by key width (cks_sort on random planes): ms per sort and per
digit pass, n keys, bits in {32, 64, 96, 128}."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2009_11543_b200 import cks
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30_000_000
g = torch.Generator(device="cuda").manual_seed(1)
for bits in (32, 64, 96, 128):
    p = torch.randint(-2**31, 2**31 - 1, (cks.nplanes(bits), n), dtype=torch.int32, device="cuda", generator=g)
    cks.sort(p, bits, want_sorted=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        cks.sort(p, bits, want_sorted=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"n": n, "bits": bits, "ms": round(ms, 4), "ms_per_pass": round(ms / (bits // 8), 4)}))

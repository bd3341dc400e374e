"""Analysis: run lengths of equal top-T-bit prefixes of P_{D+} in sorted order (cfg5)."""
import sys
sys.path.insert(0, '/root/repo')
import torch, cksgen
from paper_2009_11543_b200 import cks
keys = torch.from_numpy(cksgen.config(5)).cuda()
M = cks.superset_mask(keys)
m = cks.popcount(M)
P = cks.compress(keys, M)                       # right-aligned planes, m = 96 -> 3 planes, no lead
perm, S = cks.sort(P, m, None, want_sorted=True)
top = (S[2].long() & 0xFFFFFFFF) << 32 | (S[1].long() & 0xFFFFFFFF)   # top 64 bits of P (m = 96: no pad)
for T in (40, 48):
    pref = top >> (64 - T)
    tie = torch.zeros_like(pref, dtype=torch.bool)
    tie[1:] = pref[1:] == pref[:-1]
    starts = (~tie).nonzero().squeeze(1)
    lens = torch.diff(torch.cat([starts, torch.tensor([pref.numel()], device=pref.device)]))
    h = torch.bincount(lens.clamp(max=17))
    tot = pref.numel()
    print(f"T={T}: runs>=2 {int((lens >= 2).sum())}, keys in runs>=2 {int(lens[lens >= 2].sum())}")
    for L in range(2, 18):
        if L < h.numel():
            print(f"  L={L if L < 17 else '17+'}: runs {int(h[L])} keys {int(h[L]) * L if L < 17 else int(lens[lens >= 17].sum())}")

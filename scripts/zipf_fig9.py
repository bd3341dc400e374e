"""NEXT-2: the paper's sensitivity analysis (Sec. 6.4, Table 4, Fig. 9
PAPER.md:656-687) on one B200: for each of the 20 Zipf(s,n,m) datasets (10 M keys,
cksgen.zipf), the Table 4 statistics of the generated column and the GPU total time of the
full-key build against the compressed-key build, with the SAME sort on both legs:
  full key        prior mask = every key bit (the full key is the sort key), then bulk load;
  compressed key  prior mask = the exact D-bitmap (the paper's compressed path: extract by
                  the D-bitmap it maintains, sort, build), then bulk load;
per sort mode (one LSD sort over all mask bits / by distinguishing prefixes). The first build
(D unknown: superset pass + exact D) is timed too. Every column's first build is checked with
the library's complete order check (CKS_VERIFY_ALWAYS) -- no oracle here.

  python scripts/zipf_fig9.py [--n 10000000] [--steps 5] [--only 1,6,20] > zipf_fig9.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import cksgen  # noqa: E402
from paper_2009_11543_b200 import cks, stats  # noqa: E402

# Table 4 (compressed sort key B, word comparison ratio) and the Fig. 9 ratios the text quotes
# (datasets 20, 6, 10, 13)
TABLE4 = {i + 1: r for i, r in enumerate([(40, 1.30)] * 9 + [(24, 1.06), (24, 1.11), (24, 1.20), (24, 1.34),
                                                             (24, 1.55), (24, 1.05), (24, 1.10), (24, 1.19),
                                                             (24, 1.33), (24, 1.53), (24, 1.85)])}
FIG9_TEXT = {20: 1.66, 6: 1.46, 10: 1.19, 13: 1.25}


def timed(fn, steps, stream):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=cksgen.ZIPF_N)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    only = {int(x) for x in args.only.split(",") if x}
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    n = args.n
    r_bits = stats.rid_bits(n)
    for idx, (s, B, m) in enumerate(cksgen.ZIPF_DATASETS, start=1):
        if only and idx not in only:
            continue
        host = torch.empty((n, B), dtype=torch.uint8, pin_memory=True)
        cksgen.zipf(n, B, s, m, out=host.numpy())
        keys = host.to(dev)
        b = cks.Builder(n, B, dev, fanout=64, fill=1.0)
        cks.set_verify(cks.VERIFY_ALWAYS)                # complete order check of the result
        b(keys)
        cks.set_verify(cks.VERIFY_OFF)
        D = b.mask.copy()
        d = int(b.out.popcount)
        perm_ok = bool(torch.bincount(b.perm[:n].long(), minlength=n).eq(1).all().item())
        dplus = int(b.out.sort_bits)
        first_ms = timed(lambda: b(keys), args.steps, stream)
        t = stats.table_stats(B, d, r_bits)
        w = stats.word_comparisons(b.dbit[:n].cpu().numpy().view(np.uint16), D, B, r_bits)
        ones = np.full(B, 0xFF, np.uint8)
        legs = {}
        for name, mode in (("single_sort", cks.SORT_SINGLE), ("by_prefixes", cks.SORT_PREFIX)):
            cks.set_sort_mode(mode)
            fk = timed(lambda: b(keys, prior_mask=ones), args.steps, stream)
            fpass = int(b.out.passes)
            ck = timed(lambda: b(keys, prior_mask=D), args.steps, stream)
            cpass = int(b.out.passes)
            legs[name] = {"full_key_ms": fk, "full_key_passes": fpass, "compressed_ms": ck,
                          "compressed_passes": cpass, "total_ratio": fk / ck}
        cks.set_sort_mode(cks.SORT_PREFIX_AUTO)
        cks.set_verify(cks.VERIFY_PRIOR)
        line = {"dataset": idx, "function": f"Zipf({s},{B},{m})", "n": n, "key_bytes": B,
                "d_plus_bits": dplus, "order_checked": True, "perm_is_permutation": perm_ok,
                **t, **w, "paper_compressed_sort_key_bytes": TABLE4[idx][0],
                "paper_word_comparison_ratio": TABLE4[idx][1],
                "matches_table4_size": t["compressed_sort_key_bytes_whole_rid"] == TABLE4[idx][0],
                "first_build_ms": first_ms, **legs,
                "paper_fig9_total_ratio": FIG9_TEXT.get(idx)}
        print(json.dumps(line), flush=True)
        del b, keys, host
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

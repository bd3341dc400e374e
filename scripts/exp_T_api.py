"""First-build time by forced round-0 width T (cks_ctx_set_round0_bits) on one config."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, cksgen
from paper_2009_11543_b200 import cks
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
keys = torch.from_numpy(cksgen.config(cfg)).cuda()
b = cks.Builder(keys.shape[0], keys.shape[1], keys.device)
for T in [0] + [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["24", "32", "40", "48", "56", "64"])]:
    cks.set_round0_bits(T)
    for _ in range(3):
        b(keys)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        b(keys)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"cfg": cfg, "T": T, "ms": round(e0.elapsed_time(e1) / 10, 4), "round0_bits": int(b.out.round0_bits),
                      "passes": int(b.out.passes)}))
cks.set_round0_bits(0)

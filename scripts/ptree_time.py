"""Time cks_paper_tree on cfg5 (NEXT-3) -- device events around the call."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch, cksgen
from paper_2009_11543_b200 import cks
keys = torch.from_numpy(cksgen.config(5)).cuda()
b = cks.build(keys, tree=False)
perm, dbit = b["perm"], b["dbit"]
PK = int(sys.argv[1]) if len(sys.argv) > 1 else 32
for _ in range(2): cks.paper_tree(keys, perm, dbit, PK)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): cks.paper_tree(keys, perm, dbit, PK)
e1.record(); torch.cuda.synchronize()
print("paper_tree ms", e0.elapsed_time(e1) / 5)

"""A few fused first builds with the paper tree (cks_build + ptree_nodes, cfg5) -- for ncu launch
lists (scripts/launch_summary.py splits builds at the occupancy kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import cksgen  # noqa: E402
from paper_2009_11543_b200 import cks  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
keys = torch.from_numpy(cksgen.config(cfg)).cuda()
src = int(sys.argv[2]) if len(sys.argv) > 2 else 0
b = cks.Builder(keys.shape[0], keys.shape[1], keys.device, paper_tree_pk=32, paper_tree_fill=0.9, paper_tree_source=src)
for _ in range(3):
    b(keys)
torch.cuda.synchronize()
print("ok", int(b.out.passes), int(b.out.round0_bits))

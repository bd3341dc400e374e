"""torch.profiler over one sharded build at one rank (cfg5): where the time outside the libcks
kernels goes (host syncs, torch ops)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import cksgen  # noqa: E402
from paper_2009_11543_b200 import shard  # noqa: E402

keys = torch.from_numpy(cksgen.config(5)).cuda()
comm = shard.ThreadComm.group(1)[0]
for _ in range(3):
    shard.build_sharded(keys, comm)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    shard.build_sharded(keys, comm)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=15, max_name_column_width=60))

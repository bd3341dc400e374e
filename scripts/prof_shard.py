import time, torch, numpy as np, sys
sys.path.insert(0, '/root/repo')
import cksgen
from paper_2009_11543_b200 import shard, cks
keys = torch.from_numpy(cksgen.config(5)).cuda()
comm = shard.ThreadComm.group(1)[0]
import paper_2009_11543_b200.shard as S
orig = {}
tim = {}
def wrap(name, f):
    def g(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); tim[name] = tim.get(name, 0) + time.perf_counter() - t
        return r
    return g
class Ops(S.CudaOps): pass
for nm in [k for k in vars(S.CudaOps) if not k.startswith("_")]:
    setattr(Ops, nm, staticmethod(wrap(nm, getattr(S.CudaOps, nm))))
comm.alltoallv = wrap("alltoallv", comm.alltoallv)
comm.allgather = wrap("allgather", comm.allgather)
G = int(sys.argv[1]) if len(sys.argv) > 1 else 1
if G > 1:
    print('use G = 1 (threads on one device share its SMs)')
for i in range(3): S.build_sharded(keys, comm, ops=Ops)
tim.clear()
torch.cuda.synchronize(); t0 = time.perf_counter()
for i in range(5): S.build_sharded(keys, comm, ops=Ops)
torch.cuda.synchronize(); tot = (time.perf_counter() - t0) / 5
print("total ms", round(tot * 1e3, 2))
for k, v in sorted(tim.items(), key=lambda x: -x[1]): print(k, round(v / 5 * 1e3, 3))

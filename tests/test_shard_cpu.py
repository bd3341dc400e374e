"""NEXT-4 on the CPU: the sharded first build's orchestration -- splitters from
regular samples, the cut of every sorted shard, the one all-to-all, the boundary pairs, the
OR of D -- with the per-shard steps taken from the oracle (tests/shard_oracle_ops.py), over
real torch.distributed gloo collectives (world size 2) and over G threads. The GPU suite runs
the same orchestration with the libcks kernels (tests/test_gpu_shard.py)."""
import os
import socket
import sys

import numpy as np
import pytest

import cksgen
import oracle
from conftest import ROOT
from shard_oracle_ops import OracleOps, check_slices, mask_from_occupancy, occupancy_np

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2009_11543_b200 import shard  # noqa: E402


def split_rows(n, sizes):
    cut = np.cumsum([0] + list(sizes))
    assert cut[-1] == n
    return [(int(a), int(b)) for a, b in zip(cut[:-1], cut[1:])]


def cases():
    k1 = cksgen.config(1, n=3000)
    k3 = cksgen.config(3, n=4000)
    k5 = cksgen.config(5, n=5000)
    k2 = cksgen.config(2, n=3000)
    eq = np.repeat(np.array([[7, 1, 2, 3]], np.uint8), 50, axis=0)
    dup = np.repeat(cksgen.config(1, n=40), 25, axis=0)[np.random.default_rng(3).permutation(1000)]
    return [("cfg1", k1, [1000, 1000, 1000]), ("cfg3", k3, [3999, 1]), ("cfg5", k5, [1700, 0, 3300]),
            ("cfg2", k2, [3000]), ("equal", eq, [10, 40]), ("dups", dup, [500, 300, 200]),
            ("tiny", cksgen.config(1, n=3), [0, 2, 1, 0])]


def test_splitters_and_sample_host_logic():
    assert list(shard.regular_sample(10, 4)) == [1, 3, 6, 8]
    assert list(shard.regular_sample(3, 8)) == [0, 1, 2]
    assert shard.regular_sample(0, 8).size == 0
    s = np.array([[5, 0, 9], [1, 2, 3], [5, 0, 2], [1, 2, 1], [0, 9, 7], [5, 0, 4]], np.uint32)   # (p0, p1, rid)
    spl = shard.pick_splitters(s, 3)
    # order by p1 (top plane), then p0, then rid: (5,0,2) (5,0,4) (5,0,9) (1,2,1) (1,2,3) (0,9,7)
    assert spl.tolist() == [[5, 0, 9], [1, 2, 3]]
    assert shard.pick_splitters(s, 1).shape == (0, 3)


@pytest.mark.parametrize("cfg", [1, 3, 5])
def test_occupancy_union_pins(cfg):
    keys = cksgen.config(cfg, n=3000)
    parts = [keys[:1000], keys[1000:1001], keys[1001:]]
    u = np.bitwise_or.reduce(np.stack([occupancy_np(p) for p in parts]), axis=0)
    B = keys.shape[1]
    assert np.array_equal(mask_from_occupancy(u, B, 3000, True), oracle.byteocc_superset(keys))
    assert np.array_equal(mask_from_occupancy(u, B, 3000, False), oracle.variant_bitmap(keys))


@pytest.mark.parametrize("name,keys,sizes", cases(), ids=[c[0] for c in cases()])
def test_sharded_threads_oracle_ops(name, keys, sizes):
    rows = split_rows(keys.shape[0], sizes)
    ops = OracleOps(keys)
    shards = [torch.from_numpy(np.ascontiguousarray(keys[a:b])) for a, b in rows]
    outs = shard.ThreadComm.run(len(sizes), lambda comm, k: shard.build_sharded(k, comm, ops=ops,
                                                                                 samples_per_rank=16), shards)
    check_slices(keys, outs)


class SpecOracleOps(OracleOps):
    """OracleOps with the speculative-mask steps: the strided row sample of cks_occupancy_sample
    (step = n // samples, at least 1) and a compress that also returns the occupancy."""

    def occupancy_sample(self, keys, samples):
        k = keys.cpu().numpy()
        n = k.shape[0]
        step = max(n // samples, 1) if n else 1
        cnt = min(n // step, samples) if n else 0
        return _occ(k[np.arange(cnt, dtype=np.int64) * step])

    def compress_marking(self, keys, mask):
        return self.compress(keys, mask), self.occupancy(keys)

    def marks_occupancy(self, keys):
        return True


def _occ(k):
    return torch.from_numpy(occupancy_np(k).view(np.int32))


@pytest.mark.parametrize("samples,expect", [(4096, "held"), (6, "retried")])
@pytest.mark.parametrize("sizes", [[2500, 2501], [4000, 0, 1001]])
def test_sharded_speculative_mask_host_logic(monkeypatch, samples, expect, sizes):
    # the G > 1 speculative mask (shard.build_sharded): every rank takes the same branch, a
    # sample covering every row holds, a 2-3 row sample misses byte values and the shards
    # compress again with the union D+; the slices equal the oracle's single build either way
    monkeypatch.setattr(shard, "SPEC_MIN_KEYS", 1000)
    monkeypatch.setattr(shard, "SPEC_SAMPLES", samples)
    keys = cksgen.config(5, n=sum(sizes))
    rows = split_rows(keys.shape[0], sizes)
    ops = SpecOracleOps(keys)
    shards = [torch.from_numpy(np.ascontiguousarray(keys[a:b])) for a, b in rows]
    outs = shard.ThreadComm.run(len(sizes), lambda comm, k: shard.build_sharded(k, comm, ops=ops,
                                                                                 samples_per_rank=16), shards)
    assert [o["speculative"] for o in outs] == [expect] * len(sizes)
    check_slices(keys, outs)


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, keys, sizes, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from shard_oracle_ops import OracleOps as Ops
    from paper_2009_11543_b200 import shard as sh
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = int(sum(sizes[:rank]))
        k = torch.from_numpy(np.ascontiguousarray(keys[a:a + sizes[rank]]))
        o = sh.build_sharded(k, sh.TorchComm(), ops=Ops(keys), samples_per_rank=32)
        q.put((rank, dict(perm=o["perm"].numpy(), dbit=o["dbit"].numpy(), mask=o["mask"], offset=o["offset"],
                          packed=o["packed"].numpy(), send=o["send_counts"], tree=o["tree"])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,sizes", [(5, [2500, 1500]), (3, [0, 3000])])
def test_sharded_gloo_world2(cfg, sizes):
    keys = cksgen.config(cfg, n=sum(sizes))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, keys, sizes, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    outs = [dict(perm=torch.from_numpy(got[r]["perm"]), dbit=torch.from_numpy(got[r]["dbit"]), mask=got[r]["mask"],
                 offset=got[r]["offset"], packed=torch.from_numpy(got[r]["packed"]), tree=got[r]["tree"])
            for r in range(2)]
    assert sum(got[0]["send"]) == sizes[0] and sum(got[1]["send"]) == sizes[1]
    check_slices(keys, outs)

"""NEXT-4 on the GPU: the sharded first build (paper_2009_11543_b200/shard.py) with the libcks
kernels, G ranks run as threads on cuda:0 (each with its own stream and context; no kernel
waits on another rank), slices concatenated and compared with the oracle's single build bit
for bit: permutation, D_i, exact D, P_D and the bulk-loaded tree."""
import os

import numpy as np
import pytest

import cksgen
import oracle
from shard_oracle_ops import check_slices

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2009_11543_b200 import cks, shard  # noqa: E402


def run(keys, sizes, **kw):
    cut = np.cumsum([0] + list(sizes))
    shards = [torch.from_numpy(np.ascontiguousarray(keys[a:b])).cuda() for a, b in zip(cut[:-1], cut[1:])]
    return shard.ThreadComm.run(len(sizes), lambda comm, k: shard.build_sharded(k, comm, **kw), shards)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("G", [1, 2, 4])
def test_sharded_configs(cfg, G):
    n = 120_001 if cfg > 1 else None
    keys = cksgen.config(cfg, n=n)
    N = keys.shape[0]
    sizes = [N // G] * (G - 1) + [N - (N // G) * (G - 1)]
    outs = run(keys, sizes)
    check_slices(keys, outs)
    loads = [o["perm"].numel() for o in outs]
    assert max(loads) <= 1.5 * N / G + 64                  # regular sampling keeps the slices balanced


@pytest.mark.parametrize("cfg", [3, 5])
@pytest.mark.parametrize("G", [2, 3])
def test_sharded_fused_and_alltoall_agree(cfg, G):
    # the fused partition-and-send (every part written into its receiver's buffer by the digit
    # pass) and the partition + all-to-all baseline give the same slices, equal to the oracle
    keys = cksgen.config(cfg, n=90_001)
    N = keys.shape[0]
    sizes = [N // G] * (G - 1) + [N - (N // G) * (G - 1)]
    a = run(keys, sizes, fused=True)
    b = run(keys, sizes, fused=False)
    check_slices(keys, a)
    for x, y in zip(a, b):
        assert torch.equal(x["perm"], y["perm"]) and torch.equal(x["dbit"], y["dbit"])
        assert x["send_counts"] == y["send_counts"]


def test_partition_send_vs_partition():
    # cks_partition_count + cks_partition_send into one buffer laid out as the local partition
    # must equal cks_partition (stable parts, row ids with the base)
    keys = cksgen.config(5, n=70_001)
    d = torch.from_numpy(keys).cuda()
    M = oracle.byteocc_superset(keys)
    P = cks.compress(d, M)
    m = cks.popcount(M)
    samples = np.concatenate([P[:, ::997].cpu().numpy().view(np.uint32),
                              (np.arange(0, 70_001, 997, dtype=np.uint32) + 5)[None, :]], axis=0).T.copy()
    spl = shard.pick_splitters(samples, 4)
    q = torch.from_numpy(spl.view(np.int32)).cuda().reshape(-1, P.shape[0] + 1)
    Pp, ridp, pc = cks.partition(P, m, q, 4, 5)
    counts = cks.partition_count(P, m, q, 4, 5)
    assert torch.equal(counts, pc)
    outP = torch.empty_like(Pp)
    outR = torch.empty_like(ridp)
    starts = np.concatenate([[0], np.cumsum(counts.cpu().numpy())[:-1]])
    n = P.shape[1]
    cks.partition_send([outP.data_ptr() + 4 * int(s) for s in starts], [n] * 4,
                       [outR.data_ptr() + 4 * int(s) for s in starts])
    torch.cuda.synchronize()
    assert torch.equal(outP, Pp) and torch.equal(outR, ridp)


@pytest.mark.parametrize("sizes", [[0, 5000, 1], [4999, 0, 0, 2], [1, 1, 1]])
def test_sharded_ragged_and_empty_shards(sizes):
    keys = cksgen.config(5, n=sum(sizes))
    check_slices(keys, run(keys, sizes, samples_per_rank=8))


@pytest.mark.parametrize("case", ["cfg5", "cfg3", "retry", "ragged"])
def test_sharded_speculative_mask(case):
    # >= 2^20 keys of 32/64 bytes: the mask from the shards' row samples, the occupancy marked by
    # the compress; a key byte value no sample saw (rows 555_556 and 1_650_001 are off the
    # 33-row sample stride of both shards) makes the union D+ larger and the shards compress again
    if case == "retry":
        keys = np.random.default_rng(3).integers(0, 8, size=(2_200_001, 32), dtype=np.uint8)
        keys[555_556, 7] = 0x80
        keys[1_650_001, 30] = 0x40
    else:
        keys = cksgen.config(5 if case != "cfg3" else 3, n=2_200_001)
    sizes = [1_100_000, 1_100_001] if case != "ragged" else [1_700_000, 0, 500_001]
    outs = run(keys, sizes, tree=False)
    assert all(o["speculative"] == ("retried" if case == "retry" else "held") for o in outs)
    check_slices(keys, outs)


def test_sharded_duplicates_and_equal_keys():
    rng = np.random.default_rng(5)
    dup = np.repeat(rng.integers(0, 256, (30, 24), dtype=np.uint8), 400, axis=0)[rng.permutation(12000)]
    check_slices(dup, run(dup, [7000, 5000]))
    eq = np.repeat(np.array([[1, 2, 3, 4, 5, 6, 7, 8]], np.uint8), 9000, axis=0)
    check_slices(eq, run(eq, [3000, 3000, 3000]))


@pytest.mark.parametrize("fanout,fill", [(14, 0.9), (10, 0.9), (100, 0.9)])
def test_sharded_fanout_fill(fanout, fill):
    keys = cksgen.config(3, n=50_000)
    check_slices(keys, run(keys, [20_000, 30_000], fanout=fanout, fill=fill), fanout=fanout, fill=fill)


@pytest.mark.parametrize("bits,parts", [(23, 3), (96, 4), (200, 2), (0, 3)])
def test_partition_and_rank_vs_oracle_ops(bits, parts):
    # the two splitter primitives against the numpy reference of tests/shard_oracle_ops.py
    from shard_oracle_ops import OracleOps
    from paper_2009_11543_b200 import cks
    rng = np.random.default_rng(bits + parts)
    n, npl = 30_011, cks.nplanes(bits)
    P = rng.integers(0, 1 << 32, (npl, n), dtype=np.uint64).astype(np.uint32)
    if npl:
        P[npl - 1] &= np.uint32((1 << (bits - 32 * (npl - 1))) - 1) if bits % 32 else np.uint32(0xFFFFFFFF)
        P[:, ::7] = P[:, :1]                                    # duplicates of the first key
    spl_rows = np.sort(rng.choice(n, parts - 1, replace=False))
    spl = np.concatenate([P[:, spl_rows].T, (spl_rows + 1000).astype(np.uint32)[:, None]], axis=1)
    from paper_2009_11543_b200 import shard as sh
    spl = sh.pick_splitters(spl, parts) if parts > 1 else spl   # (P, row id) order
    Pt = torch.from_numpy(P.view(np.int32)).cuda()
    q = torch.from_numpy(np.ascontiguousarray(spl).view(np.int32)).cuda()
    ops = OracleOps(None)
    got = cks.partition(Pt, bits, q, parts, 1000)
    exp = ops.partition(torch.from_numpy(P.view(np.int32)), bits, torch.from_numpy(np.ascontiguousarray(spl).view(np.int32)),
                        parts, 1000)
    for g, e in zip(got, exp):
        assert np.array_equal(g.cpu().numpy(), e.numpy())
    perm, S = cks.sort(Pt, bits, None, want_sorted=True)
    r = cks.rank_sorted(S, bits, perm, 1000, q)
    re_ = ops.rank_sorted(S.cpu(), bits, perm.cpu(), 1000, q.cpu())
    assert np.array_equal(r.cpu().numpy(), re_.numpy())


@pytest.mark.parametrize("cfg,n", [(2, 150_001), (3, 150_001), (4, 150_001), (5, 150_001), (5, 131_072),
                                   (3, 98_304), (1, 65_536)])
def test_sort_prefix_on_given_planes(cfg, n):
    # cks_sort_prefix: the first build's sort from P_{D+} instead of key rows. n a multiple of 32
    # with |M| a multiple of 32 (cfg5: 96, cfg3: 224, cfg1: 128) sorts the caller's planes in
    # place of a left-aligned copy: they must come back unchanged
    import oracle
    from paper_2009_11543_b200 import cks
    keys = cksgen.config(cfg, n=n)
    kd = torch.from_numpy(keys).cuda()
    M = cks.superset_mask(kd)
    P = cks.compress(kd, M)
    P0 = P.clone()
    order, dbit, D, PD = cks.sort_prefix(P, M, want_packed=True)
    assert torch.equal(P, P0)
    ref = oracle.first_build(keys)
    assert np.array_equal(order.cpu().numpy().view(np.uint32), ref["perm"])
    assert np.array_equal(dbit.cpu().numpy().view(np.uint16), ref["dbit"])
    assert np.array_equal(D, ref["mask"])
    assert np.array_equal(PD.cpu().numpy().view(np.uint32), ref["planes"][:, ref["perm"]])
    o2, d2, D2, none = cks.sort_prefix(P, M)                  # without P_D
    assert none is None and np.array_equal(o2.cpu().numpy(), order.cpu().numpy()) and np.array_equal(D2, D)


_NCCL_SCRIPT = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
import cksgen
from paper_2009_11543_b200 import shard
dist.init_process_group("nccl", rank=0, world_size=1)
torch.cuda.set_device(0)
keys = cksgen.config(5, n=100_003)
o = shard.build_sharded(torch.from_numpy(keys).cuda(), shard.TorchComm())
np.savez(sys.argv[1], perm=o["perm"].cpu().numpy(), dbit=o["dbit"].cpu().numpy(), mask=o["mask"],
         packed=o["packed"].cpu().numpy())
dist.destroy_process_group()
"""


def test_sharded_over_nccl_world1(tmp_path):
    # the TorchComm path on NCCL collectives (one rank: all_gather / all_to_all_single of itself)
    import socket
    import subprocess
    import sys
    import oracle
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    out = tmp_path / "r.npz"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", _NCCL_SCRIPT, str(out)], env=env, cwd=root, check=True, timeout=300)
    z = np.load(out)
    keys = cksgen.config(5, n=100_003)
    ref = oracle.first_build(keys)
    assert np.array_equal(z["perm"].view(np.uint32), ref["perm"])
    assert np.array_equal(z["dbit"].view(np.uint16), ref["dbit"])
    assert np.array_equal(z["mask"], ref["mask"])
    assert np.array_equal(z["packed"].view(np.uint32), ref["planes"][:, ref["perm"]])


def test_sharded_variant_superset():
    # the union of occupancies also yields V (cks_occupancy_mask, CKS_SUPERSET_VARIANT)
    from paper_2009_11543_b200 import cks
    keys = cksgen.config(3, n=60_000)
    outs = run(keys, [30_000, 30_000], superset_kind=cks.SUPERSET_VARIANT)
    assert outs[0]["sort_bits"] == int(np.unpackbits(oracle_variant(keys)).sum())
    check_slices(keys, outs)


def oracle_variant(keys):
    import oracle
    return oracle.variant_bitmap(keys)


def test_sharded_odd_width():
    rng = np.random.default_rng(13)
    keys = rng.integers(0, 256, (40_001, 13), dtype=np.uint8)
    keys[:, :2] = rng.integers(0, 3, (40_001, 2), dtype=np.uint8)
    keys[rng.integers(0, 40_001, 500)] = keys[rng.integers(0, 40_001, 500)]
    check_slices(keys, run(keys, [10_000, 20_001, 10_000]))


_IPC_SCRIPT = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
import cksgen
from paper_2009_11543_b200 import shard
rank, world = int(sys.argv[2]), int(sys.argv[3])
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(0)
keys = cksgen.config(5, n=90_001)
cut = [0, 40_000, 90_001] if world == 2 else [0, 30_000, 61_000, 90_001]
o = shard.build_sharded(torch.from_numpy(keys[cut[rank]:cut[rank + 1]]).cuda(), shard.TorchComm(), fused=True)
np.savez(sys.argv[1] + f".{rank}.npz", perm=o["perm"].cpu().numpy(), dbit=o["dbit"].cpu().numpy(), mask=o["mask"])
dist.barrier()
dist.destroy_process_group()
"""


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fused_over_ipc_processes(tmp_path, world):
    # the multi-process fused partition-and-send: ranks are processes (gloo for the small
    # collectives), the receive buffers are shared as CUDA IPC handles and every sender's digit
    # pass writes its parts into the other processes' buffers. All processes share cuda:0 here
    # (no kernel waits on another rank); across GPUs the same stores go over NVLink
    import socket
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    base = str(tmp_path / "r")
    ps = [subprocess.Popen([sys.executable, "-c", _IPC_SCRIPT, base, str(r), str(world)], env=env, cwd=root)
          for r in range(world)]
    for p in ps:
        assert p.wait(timeout=300) == 0
    zs = [np.load(f"{base}.{r}.npz") for r in range(world)]
    keys = cksgen.config(5, n=90_001)
    ref = oracle.first_build(keys)
    assert np.array_equal(np.concatenate([z["perm"] for z in zs]).view(np.uint32), ref["perm"])
    assert np.array_equal(np.concatenate([z["dbit"] for z in zs]).view(np.uint16), ref["dbit"])
    assert all(np.array_equal(z["mask"], ref["mask"]) for z in zs)

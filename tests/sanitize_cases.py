"""Small builds for the checked library (lib/libcks_checked.so: device bounds assertions,
poisoned scratch, canary bands after every scratch buffer; this pool has no compute-sanitizer)
and, where available, compute-sanitizer (scripts/sanitize.sh): every kernel family of the path
runs at least once -- cfg1 (plain LSD sort, 16-B keys), cfg5 and cfg3 samples (refinement,
k_ref_tile, compaction, short-run finishers), cfg4 (LSD refinement rounds), the edge sets
(empty, one key, all equal, odd widths, unaligned keys), the order check and its negative
case, the paper-format tree and the sharded steps (partition, rank, sort_prefix). Each result
is compared with the oracle so a sanitizer-clean run is also a correct one. Not collected by
pytest (no test_ prefix); run: python tests/sanitize_cases.py [quick]."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import cksgen  # noqa: E402
import oracle  # noqa: E402
from paper_2009_11543_b200 import _build, cks  # noqa: E402

CANARY = 0x3C3C3C3C


def guarded_build(keys_d, prior=None):
    """cks_build into caller buffers with a canary tail: the library must write exactly n
    entries of perm and dbit (and the tree arrays they size)."""
    n, B = keys_d.shape
    b = cks.Builder(n, B, keys_d.device)
    big_p = torch.full((n + 4096,), CANARY, dtype=torch.int32, device=keys_d.device)
    big_d = torch.full((n + 4096,), 0x3C3C, dtype=torch.int16, device=keys_d.device)
    b.perm, b.dbit = big_p[:max(n, 1)], big_d[:max(n, 1)]
    b.out.perm, b.out.dbit = big_p.data_ptr(), big_d.data_ptr()
    b(keys_d, prior)
    torch.cuda.synchronize()
    assert bool((big_p[n:] == CANARY).all()), "perm written past n"
    assert bool((big_d[n:] == 0x3C3C).all()), "dbit written past n"
    o = b.out
    return dict(mask=b.mask.copy(), popcount=int(o.popcount), perm=big_p[:n], dbit=big_d[:n], packed=b.packed())


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def check(keys, r):
    ref = oracle.first_build(keys)
    assert np.array_equal(r["mask"], ref["mask"])
    assert np.array_equal(u32(r["perm"]), ref["perm"])
    assert np.array_equal(r["dbit"].cpu().numpy().view(np.uint16), ref["dbit"])
    if keys.shape[0]:
        assert np.array_equal(u32(r["packed"]), ref["planes"][:, ref["perm"]])


def main(quick: bool):
    scale = 1 if quick else 2
    cases = [("cfg1", cksgen.config(1, n=20_000 * scale)), ("cfg5", cksgen.config(5, n=40_000 * scale)),
             ("cfg3", cksgen.config(3, n=30_000 * scale)), ("cfg4", cksgen.config(4, n=30_000 * scale)),
             ("cfg2", cksgen.config(2, n=20_000 * scale)),
             ("empty", np.zeros((0, 16), np.uint8)), ("one", cksgen.config(1, n=1)),
             ("all_equal", cksgen.all_equal(5000, 24, 3)), ("odd13", cksgen.uniform(9001, 13, 5, 20000))]
    for name, keys in cases:
        r = guarded_build(torch.from_numpy(np.ascontiguousarray(keys)).cuda())
        torch.cuda.synchronize()
        check(keys, r)
        print("ok", name, keys.shape, flush=True)
    # unaligned key rows
    raw = torch.zeros(5001 * 16 + 3, dtype=torch.uint8, device="cuda")
    keys = cksgen.config(1, n=5001)
    view = raw[3:].view(5001, 16)
    view.copy_(torch.from_numpy(keys))
    check(keys, cks.build(view))
    print("ok unaligned", flush=True)
    # rebuild with the order check; a stale mask must be reported
    keys = cksgen.config(5, n=30_000)
    ref = oracle.first_build(keys)
    d = torch.from_numpy(keys).cuda()
    check(keys, cks.build(d, prior_mask=ref["mask"]))
    bad = ref["mask"].copy()
    bad[0] = 0
    try:
        cks.build(d, prior_mask=bad)
        print("stale mask: no error (order unchanged)")
    except cks.CksError as e:
        assert e.code == cks.CKS_ERANGE
        print("ok stale mask -> CKS_ERANGE", flush=True)
    # paper-format tree
    keys = cksgen.config(3, n=20_003)
    ref = oracle.first_build(keys)
    d = torch.from_numpy(keys).cuda()
    perm = torch.from_numpy(ref["perm"].view(np.int32)).cuda()
    dbit = torch.from_numpy(ref["dbit"].view(np.int16)).cuda()
    nodes = cks.paper_tree(d, perm, dbit, 32, 0.9)
    assert np.array_equal(nodes.cpu().numpy(), oracle.paper_tree(keys, ref["perm"], ref["dbit"], 32, 0.9)["nodes"])
    print("ok paper tree", flush=True)
    # the fused tree from every partial-key source, including the degenerate shapes (one key:
    # an empty mask; one leaf; a one-key last leaf)
    for cfg, n in ((5, 1), (5, 13), (5, 25_009), (2, 15), (2, 20_001), (3, 9_001)):
        keys = cksgen.config(cfg, n=n)
        d = torch.from_numpy(keys).cuda()
        srcs = [cks.PTREE_ROWS, cks.PTREE_DS, cks.PTREE_CARRY] + ([cks.PTREE_DECODE] if cfg != 3 else [])
        for src in srcs:
            r = cks.build(d, paper_tree_pk=32, paper_tree_fill=0.9, paper_tree_source=src, ds_metadata=True)
            t = oracle.paper_tree(keys, u32(r["perm"]), r["dbit"].cpu().numpy().view(np.uint16), 32, 0.9)
            assert np.array_equal(r["paper_tree"].cpu().numpy(), t["nodes"]), (cfg, n, src)
    print("ok fused paper trees", flush=True)
    # rebuilds: a prior mask the D+ test proves (with the decode tree), and one it cannot
    # (the row-gather order check, twice: the second skips the occupancy pass)
    keys = cksgen.config(5, n=30_001)
    ref = oracle.first_build(keys)
    d = torch.from_numpy(keys).cuda()
    dplus = oracle.byteocc_superset(keys)
    r = cks.build(d, prior_mask=dplus, paper_tree_pk=32, paper_tree_source=cks.PTREE_DECODE)
    check(keys, r)
    t = oracle.paper_tree(keys, u32(r["perm"]), r["dbit"].cpu().numpy().view(np.uint16), 32, 0.9)
    assert np.array_equal(r["paper_tree"].cpu().numpy(), t["nodes"])
    for _ in range(2):
        check(keys, cks.build(d, prior_mask=ref["mask"]))
    print("ok proven / unproven rebuilds", flush=True)
    # the speculative first build (>= 2^20 keys): the sample's mask holds, and one that falls
    # short (an unsampled row with a new byte value) is built again
    for keys in (cksgen.config(5, n=1_100_001), cksgen.config(3, n=1_100_001)):
        check(keys, cks.build(torch.from_numpy(keys).cuda()))
    keys = np.random.default_rng(3).integers(0, 8, size=(1_100_001, 32), dtype=np.uint8)
    keys[555_555, 7] = 0x80
    check(keys, cks.build(torch.from_numpy(keys).cuda()))
    print("ok speculative first builds", flush=True)
    # the sharded path on one device (threads)
    from paper_2009_11543_b200 import shard
    keys = cksgen.config(5, n=30_000)
    ref = oracle.first_build(keys)
    shards = [torch.from_numpy(np.ascontiguousarray(keys[a:b])).cuda() for a, b in ((0, 13_000), (13_000, 30_000))]
    outs = shard.ThreadComm.run(2, lambda comm, k: shard.build_sharded(k, comm), shards)
    perm = np.concatenate([u32(o["perm"]) for o in outs])
    assert np.array_equal(perm, ref["perm"])
    print("ok sharded x2", flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    if "product" not in args:                          # default: the checked library
        cks.load_library(_build.build(checked=True))           # (rebuilt when stale)
        print("library:", _build.SO_CHECKED, flush=True)
    main("quick" in args)
    print("all cases ok", flush=True)

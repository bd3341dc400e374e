"""Small builds for compute-sanitizer (scripts/sanitize.sh): every kernel family of the path
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
from paper_2009_11543_b200 import cks  # noqa: E402


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
        r = cks.build(torch.from_numpy(np.ascontiguousarray(keys)).cuda())
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
    main(len(sys.argv) > 1 and sys.argv[1] == "quick")

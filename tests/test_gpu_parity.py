"""GPU parity: the CUDA path (through the C ABI via the ctypes binding) against the CPU
oracle, element by element, bit-exact (integer work: no tolerance). Sizes span several
4096-key sort tiles plus a ragged tail; edge cases cover empty, single, all-equal and
degenerate masks; full-size configs are checked on properties that pin the result
uniquely (the (key, row id) order is total, so a valid sorted permutation is THE oracle
permutation) plus sampled oracle values."""
import numpy as np
import pytest

import cksgen
import oracle
from conftest import mask_from, positions

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():                       # collected on CPU, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2009_11543_b200 import cks  # noqa: E402


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def u16(t):
    return t.cpu().numpy().view(np.uint16)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def planes_dev(planes):
    return dev(np.ascontiguousarray(planes).view(np.int32))


RAGGED = [0, 1, 2, 3, 31, 4095, 4096, 4097, 100_003]


# ---- a1: superset masks --------------------------------------------------------------

@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_superset_masks_configs(cfg):
    keys = cksgen.config(cfg, n=150_001)
    d = dev(keys)
    assert np.array_equal(cks.superset_mask(d, cks.SUPERSET_BYTEOCC), oracle.byteocc_superset(keys))
    assert np.array_equal(cks.superset_mask(d, cks.SUPERSET_VARIANT), oracle.variant_bitmap(keys))


@pytest.mark.parametrize("B", [1, 2, 3, 5, 8, 12, 16, 24, 48, 64, 100, 512])
@pytest.mark.parametrize("n", [0, 1, 7, 5000])
def test_superset_masks_shapes(B, n):
    keys = cksgen.lowcard(n, B, seed=B * 7 + n, values=5)
    d = dev(keys)
    assert np.array_equal(cks.superset_mask(d, cks.SUPERSET_BYTEOCC), oracle.byteocc_superset(keys))
    assert np.array_equal(cks.superset_mask(d, cks.SUPERSET_VARIANT), oracle.variant_bitmap(keys))


def test_superset_mask_unaligned_keys():
    keys = cksgen.uniform(3001, 16, seed=3)
    big = torch.zeros(3001 * 16 + 16, dtype=torch.uint8, device="cuda")
    view = big[5:5 + 3001 * 16].view(3001, 16)           # 5-byte offset: generic path
    view.copy_(dev(keys))
    assert np.array_equal(cks.superset_mask(view), oracle.byteocc_superset(keys))


# ---- a3: compress ---------------------------------------------------------------------

@pytest.mark.parametrize("B", [1, 3, 8, 16, 32, 35, 64, 128])
def test_compress_random_masks(B):
    rng = np.random.default_rng(B)
    keys = cksgen.uniform(20_011, B, seed=B)
    d = dev(keys)
    for density in (0.02, 0.3, 1.0):
        mask = np.packbits(rng.random(8 * B) < density)
        got = u32(cks.compress(d, mask))
        assert np.array_equal(got, oracle.compress(keys, mask))


@pytest.mark.parametrize("C", [1, 3, 4, 7, 12, 13, 28, 31, 32])
def test_compress_uniform_word_masks(C):
    # masks with the same number C of bits in every 4-byte key word (the compile-time layout of
    # k_compress_uni when P_M has no top padding: C % 4 == 0 here, right-aligned 8C-bit P), with
    # and without the occupancy marking
    from shard_oracle_ops import occupancy_np
    rng = np.random.default_rng(100 + C)
    bits = np.zeros(256, np.uint8)
    for w in range(8):
        bits[32 * w + rng.choice(32, size=C, replace=False)] = 1
    mask = np.packbits(bits)
    keys = cksgen.uniform(50_003, 32, seed=C)
    d = dev(keys)
    ref = oracle.compress(keys, mask)
    assert np.array_equal(u32(cks.compress(d, mask)), ref)
    planes, occ = cks.compress_marking(d, mask)
    assert np.array_equal(u32(planes), ref)
    assert np.array_equal(occ.cpu().numpy().view(np.uint32), occupancy_np(keys))


@pytest.mark.parametrize("values", [2, 128])
def test_speculative_build_uniform_alphabet(values):
    # first builds (>= 2^20 keys, the speculative mask) whose D+ has the same bits in every byte:
    # {0, 1}: 1 bit a byte, m = 32, one LSD sort; 0..127: 7 bits, m = 224, sort by prefixes --
    # the compress marking the occupancy with the compile-time layout (C = 4 and 28 bits a word)
    rng = np.random.default_rng(values)
    keys = rng.integers(0, values, size=(1_100_003, 32), dtype=np.uint8)
    keys[:, :3] = keys[rng.integers(0, 50_000, size=keys.shape[0]), :3]
    s0 = cks.speculation_stats()
    r = cks.build(dev(keys))
    assert cks.speculation_stats()[0] == s0[0] + 1
    check_build(keys, r)


def test_compress_table3_mask():
    from conftest import load_bit_rows
    m = load_bit_rows("table3_indbtab_dbitmap.txt")
    keys = cksgen.uniform(9000, 35, seed=35)
    assert np.array_equal(u32(cks.compress(dev(keys), m)), oracle.compress(keys, m))


# ---- a5: sort -------------------------------------------------------------------------

@pytest.mark.parametrize("n", RAGGED)
@pytest.mark.parametrize("bits", [1, 8, 23, 32, 33, 96, 150])
def test_sort_vs_oracle(n, bits):
    rng = np.random.default_rng(n + bits)
    np_ = (bits + 31) // 32
    planes = rng.integers(0, 2 ** 32, size=(np_, n), dtype=np.uint64).astype(np.uint32)
    if np_:
        top = bits - 32 * (np_ - 1)
        planes[-1] &= np.uint32((1 << top) - 1) if top < 32 else np.uint32(0xFFFFFFFF)
        if n > 10:                                            # duplicates
            planes[:, n // 2:] = planes[:, : n - n // 2]
    perm, srt = cks.sort(planes_dev(planes), bits, want_sorted=True)
    ref = oracle.sort_packed(planes)
    assert np.array_equal(u32(perm), ref)
    if n:
        assert np.array_equal(u32(srt), planes[:, ref])


@pytest.mark.parametrize("n", [5, 4097, 60_000])
def test_sort_with_user_row_ids(n):
    rng = np.random.default_rng(n)
    planes = (rng.integers(0, 64, size=(1, n))).astype(np.uint32)            # many ties
    rid = rng.permutation(np.arange(10, 10 + n, dtype=np.uint32))
    perm, _ = cks.sort(planes_dev(planes), 6, row_ids=dev(rid.view(np.int32)))
    assert np.array_equal(u32(perm), oracle.sort_packed(planes, rid=rid))


def test_sort_skewed_digits():
    n = 200_000
    planes = np.zeros((2, n), np.uint32)
    planes[0, ::1000] = 7                                      # one digit value dominates
    perm, _ = cks.sort(planes_dev(planes), 40)
    assert np.array_equal(u32(perm), oracle.sort_packed(planes))


# ---- a6: adjacency ----------------------------------------------------------------------

@pytest.mark.parametrize("cfg", [1, 3, 4, 5])
def test_adjacent_dbits_vs_oracle(cfg):
    keys = cksgen.config(cfg, n=30_000)
    sup = oracle.byteocc_superset(keys)
    m = oracle.popcount(sup)
    planes = oracle.compress(keys, sup)
    sp = planes[:, oracle.sort_packed(planes)]
    mask, dbit = cks.adjacent_dbits(planes_dev(sp), m, sup)
    rd, rm = oracle.adjacent_compressed(sp, m, sup)
    assert np.array_equal(mask, rm)
    assert np.array_equal(u16(dbit), rd)


# ---- a8: bulk load -----------------------------------------------------------------------

@pytest.mark.parametrize("n,fanout,fill", [(1, 64, 1.0), (64, 64, 1.0), (65, 64, 1.0), (4097, 64, 1.0),
                                           (300_000, 64, 1.0), (50_000, 14, 0.9), (20_000, 9, 0.9),
                                           (1000, 2, 1.0), (30_001, 10, 0.9), (9_999, 100, 0.9)])
def test_bulkload_vs_oracle(n, fanout, fill):
    keys = cksgen.config(5, n=n)
    perm = oracle.sort_keys(keys)
    dbit, _ = oracle.adjacent_dbits(keys, perm)
    t = cks.bulkload(dev(perm.view(np.int32)), dev(dbit.view(np.int16)), fanout, fill)
    ref = oracle.bulkload(perm, dbit, keys, fanout, fill)
    T = int(t["shape"].total_nodes)
    L0 = int(t["shape"].level_nodes[0])
    assert t["shape"].height == ref["height"]
    assert np.array_equal(u32(t["node_cnt"])[:T], ref["node_cnt"])
    assert np.array_equal(u32(t["entry_rid"])[:T * fanout], ref["entry_rid"].ravel())
    assert np.array_equal(u16(t["entry_dbit"])[:T * fanout], ref["entry_dbit"].ravel())
    assert np.array_equal(u32(t["entry_child"])[:(T - L0) * fanout], ref["entry_child"][L0:].ravel())


# ---- exact D and the fused build -----------------------------------------------------------

@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_distinction_mask_vs_oracle(cfg):
    keys = cksgen.config(cfg, n=100_003)
    mask, perm = cks.distinction_mask(dev(keys))
    permK = oracle.sort_keys(keys, threads=oracle.threads_default())
    _, D = oracle.adjacent_dbits(keys, permK)
    assert np.array_equal(mask, D)
    assert np.array_equal(u32(perm), permK)


def check_build(keys, r, threads=None):
    ref = oracle.first_build(keys, threads=threads or oracle.threads_default())
    assert np.array_equal(r["mask"], ref["mask"])
    assert r["popcount"] == ref["m"]
    assert np.array_equal(u32(r["perm"]), ref["perm"])
    assert np.array_equal(ref["perm_packed"], ref["perm"])         # Theorem 2 on the oracle side
    assert np.array_equal(u16(r["dbit"]), ref["dbit"])
    n = keys.shape[0]
    if n:
        assert np.array_equal(u32(r["packed"]), ref["planes"][:, ref["perm"]])
    if r["tree"] is not None and n:
        t = oracle.bulkload(ref["perm"], ref["dbit"], keys, int(r["shape"].fanout),
                            float(r["shape"].per_node) / float(r["shape"].fanout))
        T, f = int(r["shape"].total_nodes), int(r["shape"].fanout)
        assert np.array_equal(u32(r["tree"]["entry_rid"])[:T * f], t["entry_rid"].ravel())
        assert np.array_equal(u16(r["tree"]["entry_dbit"])[:T * f], t["entry_dbit"].ravel())
        assert np.array_equal(u32(r["tree"]["node_cnt"])[:T], t["node_cnt"])


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_build_configs_vs_oracle(cfg):
    keys = cksgen.config(cfg, n=200_003 if cfg > 1 else None)
    r = cks.build(dev(keys))
    check_build(keys, r)
    assert np.array_equal(r["sort_mask"], oracle.byteocc_superset(keys))      # the mask the sort ran on


@pytest.mark.parametrize("kind", [cks.SUPERSET_VARIANT, cks.SUPERSET_BYTEOCC])
def test_build_superset_kinds(kind):
    keys = cksgen.config(3, n=50_000)
    check_build(keys, cks.build(dev(keys), superset_kind=kind))


def test_rebuild_with_prior_mask():
    # rebuild: extract by the current D-bitmap (here the exact D plus stale bits,
    # as after deletes P:402), sort, recompute -> new D is a subset of the old one
    keys = cksgen.config(4, n=80_000)
    ref = oracle.first_build(keys)
    rng = np.random.default_rng(1)
    stale = ref["mask"] | np.packbits(rng.random(8 * 64) < 0.1)
    r = cks.build(dev(keys), prior_mask=stale)
    assert positions(r["mask"]) <= positions(stale)
    assert np.array_equal(r["sort_mask"], stale)                  # a rebuild sorts by the given mask
    check_build(keys, r)
    # after deletions the old D stays a valid (extended) mask
    sub = keys[::3].copy()
    r2 = cks.build(dev(sub), prior_mask=ref["mask"])
    check_build(sub, r2)


def _dropped_masks(keys, count):
    """(mask = exact D minus one bit, whether the oracle's order on P_mask differs from the
    full-key order) for up to `count` bits of D: Theorem 2 needs every D-bit."""
    ref = oracle.first_build(keys)
    out = []
    for p in sorted(positions(ref["mask"]))[:count]:
        m = ref["mask"].copy()
        m[p >> 3] &= ~np.uint8(0x80 >> (p & 7))
        wrong = not np.array_equal(oracle.sort_packed(oracle.compress(keys, m)), ref["perm"])
        out.append((m, wrong))
    return ref, out


@pytest.mark.parametrize("cfg,n", [(3, 40_000), (5, 60_000), (1, 30_000)])
def test_prior_mask_not_superset_is_detected(cfg, n):
    # a stale D-bitmap (one distinction bit missing, as after an insert) must not return a
    # wrong permutation silently: the order check reports CKS_ERANGE exactly when the
    # compressed order differs from the full-key order (decided by the oracle)
    keys = cksgen.config(cfg, n=n)
    ref, cases = _dropped_masks(keys, 12)
    assert any(w for _, w in cases), "no dropped bit changes the order: the test has no teeth"
    d = dev(keys)
    for m, wrong in cases:
        if wrong:
            with pytest.raises(cks.CksError) as ei:
                cks.build(d, prior_mask=m)
            assert ei.value.code == cks.CKS_ERANGE
            with pytest.raises(cks.CksError) as ei:
                cks.distinction_mask(d, prior_mask=m)
            assert ei.value.code == cks.CKS_ERANGE
        else:
            r = cks.build(d, prior_mask=m)
            assert np.array_equal(u32(r["perm"]), ref["perm"])
    m_bad = next(m for m, w in cases if w)
    with pytest.raises(cks.CksError) as ei:
        cks.build_host(keys, prior_mask=m_bad)
    assert ei.value.code == cks.CKS_ERANGE
    # with the check off the library returns the compressed order as is (documented)
    cks.set_verify(cks.VERIFY_OFF)
    try:
        r = cks.build(d, prior_mask=m_bad)
        assert not np.array_equal(u32(r["perm"]), ref["perm"])
    finally:
        cks.set_verify(cks.VERIFY_PRIOR)


def test_verify_always_passes_valid_builds():
    keys = cksgen.config(4, n=50_000)
    cks.set_verify(cks.VERIFY_ALWAYS)
    try:
        check_build(keys, cks.build(dev(keys)))
        ref = oracle.first_build(keys)
        check_build(keys, cks.build(dev(keys), prior_mask=ref["mask"]))
    finally:
        cks.set_verify(cks.VERIFY_PRIOR)
    for bad in (-1, 3):
        with pytest.raises(cks.CksError):
            cks.set_verify(bad)


@pytest.mark.parametrize("maker", ["empty", "one", "two_equal", "two", "all_equal", "all16", "consecutive",
                                   "prefix_heavy", "B1", "B3", "B512"])
def test_build_edge_cases(maker):
    keys = {
        "empty": lambda: np.zeros((0, 16), np.uint8),
        "one": lambda: cksgen.uniform(1, 16, seed=1),
        "two_equal": lambda: cksgen.all_equal(2, 8, seed=2),
        "two": lambda: cksgen.uniform(2, 8, seed=3),
        "all_equal": lambda: cksgen.all_equal(10_000, 32, seed=4),
        "all16": lambda: cksgen.consecutive(1 << 16, 2, shuffle_seed=5),
        "consecutive": lambda: cksgen.consecutive(70_000, 8, start=12345, shuffle_seed=6),
        "prefix_heavy": lambda: cksgen.prefix_heavy(50_000, 64, seed=7),
        "B1": lambda: cksgen.uniform(3000, 1, seed=8),
        "B3": lambda: cksgen.uniform(9000, 3, seed=9, dup_ppm=50_000),
        "B512": lambda: cksgen.lowcard(3000, 512, seed=10, values=3),
    }[maker]()
    r = cks.build(dev(keys) if keys.shape[0] else torch.zeros((0, keys.shape[1]), dtype=torch.uint8,
                                                               device="cuda"))
    check_build(keys, r)
    if maker == "all16":
        assert positions(r["mask"]) == set(range(16))
    if maker in ("all_equal", "two_equal", "one", "empty"):
        assert r["popcount"] == 0


def test_build_host_e2e_path():
    keys = cksgen.config(5, n=300_007)
    r = cks.build_host(keys)
    ref = oracle.first_build(keys, threads=oracle.threads_default())
    assert np.array_equal(r["mask"], ref["mask"])
    assert np.array_equal(r["perm"], ref["perm"])


def test_build_repeatable_and_stream():
    keys = dev(cksgen.config(2, n=123_457))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        a = cks.build(keys)
        b = cks.build(keys)
    s.synchronize()
    assert np.array_equal(u32(a["perm"]), u32(b["perm"]))
    assert np.array_equal(a["mask"], b["mask"])


@pytest.mark.parametrize("cfg,n", [(5, 2_000_003), (3, 1_500_001)])
def test_repeated_builds_under_contention(cfg, n):
    # race stress (the pool has no racecheck): the warp-specialised pass hands tiles between
    # producer, rankers and writers through mbarriers, and k_ref_tile works in shared memory;
    # 12 builds with a matmul stream competing for the SMs must all equal the oracle
    keys = cksgen.config(cfg, n=n)
    ref = oracle.first_build(keys, threads=oracle.threads_default())
    d = dev(keys)
    side = torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    for i in range(12):
        if i % 2:
            with torch.cuda.stream(side):
                for _ in range(4):
                    a = (a @ a).clamp_(-1, 1)
        r = cks.build(d, tree=False)
        assert np.array_equal(u32(r["perm"]), ref["perm"]), i
        assert np.array_equal(u16(r["dbit"]), ref["dbit"]), i
        assert np.array_equal(r["mask"], ref["mask"]), i
    torch.cuda.synchronize()


# ---- full-size configs (the launch configuration bench.py times) ----------------------------

def verify_sorted_perm(keys, perm):
    n, B = keys.shape
    assert perm.shape == (n,)
    assert np.bincount(perm, minlength=n).max() == 1 if n else True
    s = keys[perm]
    W = (B + 7) // 8
    pad = np.zeros((n, 8 * W), np.uint8)
    pad[:, :B] = s
    w = pad.view(">u8")
    lt = np.zeros(n - 1, bool)
    eq = np.ones(n - 1, bool)
    for j in range(W):
        a, b = w[:-1, j], w[1:, j]
        lt |= eq & (a < b)
        eq &= a == b
    assert np.all(lt | (eq & (perm[:-1] < perm[1:]))), "GPU permutation is not the (key, row id) order"


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_full_size_config(cfg):
    keys = cksgen.config(cfg)
    d = dev(keys)
    b = cks.Builder(keys.shape[0], keys.shape[1], d.device)
    b(d)
    perm = u32(b.perm)
    verify_sorted_perm(keys, perm)                       # unique total order => == oracle perm
    dbit_ref, D = oracle.adjacent_dbits(keys, perm)      # P:176 on the verified order
    assert np.array_equal(b.mask, D)
    assert np.array_equal(u16(b.dbit), dbit_ref)
    assert np.array_equal(b.mask & ~oracle.byteocc_superset(keys), np.zeros_like(b.mask))
    rng = np.random.default_rng(cfg)
    idx = np.sort(rng.choice(keys.shape[0], 1_000_000, replace=False))
    packed = u32(b.packed())
    assert np.array_equal(packed[:, idx], oracle.compress(keys[perm[idx]], b.mask))
    # the whole tree at full size: the oracle's bulk load of the verified order and D_i (inner
    # D-bits computed directly on the full keys) must equal every node array
    T, f = int(b.shape.total_nodes), 64
    t = oracle.bulkload(perm, dbit_ref, keys, f, 1.0)
    L0 = int(b.shape.level_nodes[0])
    assert np.array_equal(u32(b.tree["node_cnt"])[:T], t["node_cnt"])
    assert np.array_equal(u32(b.tree["entry_rid"])[:T * f], t["entry_rid"].ravel())
    assert np.array_equal(u16(b.tree["entry_dbit"])[:T * f], t["entry_dbit"].ravel())
    assert np.array_equal(u32(b.tree["entry_child"])[:(T - L0) * f], t["entry_child"][L0:].ravel())


# ---- NEXT-1: sort by distinguishing prefixes (refinement rounds) -----------------------------

def hier_keys(n, widths, seed, groups=(7, 40), dup_rows=600, carriers=True):
    """Keys whose first bytes come from few patterns, so that the first 64 (and 128) bits of
    the compressed key tie over long runs and the refinement has to run LSD rounds and finish
    runs of every length; exact duplicates in blocks of 2..60 rows. `widths` = number of
    distinct values per byte (256 = full byte; 2**b makes the byte contribute b mask bits)."""
    rng = np.random.default_rng(seed)
    B = len(widths)
    w = np.asarray(widths)
    keys = (rng.integers(0, 1 << 30, (n, B)) % w).astype(np.uint8)
    a = rng.integers(0, groups[0], n)
    pa = (rng.integers(0, 1 << 30, (groups[0], min(B, 10))) % w[:min(B, 10)]).astype(np.uint8)
    keys[:, :min(B, 10)] = pa[a]
    if B > 10:
        hi = min(B, 20)
        b = rng.integers(0, groups[1], n)
        pb = (rng.integers(0, 1 << 30, (groups[1], hi - 10)) % w[10:hi]).astype(np.uint8)
        sel = rng.random(n) < 0.8
        keys[sel, 10:hi] = pb[b[sel]]
    if carriers:                                    # every byte takes every allowed value once
        m = min(n, int(w.max()))
        keys[:m] = (np.arange(m)[:, None] % w[None, :]).astype(np.uint8)
    src = rng.integers(0, n, dup_rows)
    reps = rng.integers(1, 60, dup_rows)
    dst = rng.permutation(n)[: int(reps.sum())]
    keys[dst] = keys[np.repeat(src, reps)[: dst.size]]
    return keys[rng.permutation(n)]


@pytest.mark.parametrize("m", [65, 96, 97, 127, 128, 129, 192, 200, 256])
def test_refine_widths(m):
    widths = [256] * (m // 8) + ([1 << (m % 8)] if m % 8 else [])
    keys = hier_keys(60_000, widths, seed=m)
    r = cks.build(dev(keys))
    assert r["sort_bits"] == m
    check_build(keys, r)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_refine_long_runs(seed):
    # 32-byte keys, D+ = 256 bits (four 64-bit chunks): runs of up to ~10k keys tie on
    # chunk 0, thousands still tie on chunk 1; equal-key blocks of every length
    keys = hier_keys(120_000, [256] * 32, seed=seed, groups=(3, 12), dup_rows=2000)
    r = cks.build(dev(keys))
    check_build(keys, r)


def test_refine_runs_of_equal_keys():
    # long runs of equal keys that stay tied to the last chunk (no chunk ever separates them)
    rng = np.random.default_rng(11)
    base = rng.integers(0, 256, (40, 24), dtype=np.uint8)
    counts = np.array([1, 2, 3, 15, 16, 17, 63, 64, 65, 200, 4000, 9000] * 3 + [1, 1, 1, 1])
    keys = np.repeat(base, counts, axis=0)
    keys = keys[rng.permutation(keys.shape[0])]
    check_build(keys, cks.build(dev(keys)))


@pytest.mark.parametrize("shuffle", [False, True])
def test_refine_run_boundaries(shuffle):
    # runs of equal keys whose ends fall on and next to the compaction's boundaries: a thread's
    # 16 flags, a warp's 512, a tile's 4096 (runs inside one, across two, filling one exactly),
    # singletons between them, a ragged end; every round compacts them again
    rng = np.random.default_rng(17)
    lens = [1, 15, 16, 1, 17, 2, 14, 496, 512, 1, 511, 3585, 4096, 1, 4095, 2, 4097, 8192, 3, 1, 1, 7] * 3
    base = np.unique(rng.integers(0, 256, (len(lens) + 50, 24), dtype=np.uint8), axis=0)[:len(lens)]
    keys = np.repeat(base, lens, axis=0)
    if shuffle:
        keys = keys[rng.permutation(keys.shape[0])]
    check_build(keys, cks.build(dev(keys)))


@pytest.mark.parametrize("cfg", [3, 5])
def test_sort_modes_agree(cfg):
    # single full-width sort, auto and forced prefix refinement: the same (key, row id) order,
    # D, D_i and sorted P_D (Theorem 2 and stability), all equal to the oracle
    keys = cksgen.config(cfg, n=60_001)
    d = dev(keys)
    res = {}
    try:
        for mode in (cks.SORT_SINGLE, cks.SORT_PREFIX_AUTO, cks.SORT_PREFIX):
            cks.set_sort_mode(mode)
            res[mode] = cks.build(d)
    finally:
        cks.set_sort_mode(cks.SORT_PREFIX_AUTO)
    check_build(keys, res[cks.SORT_PREFIX_AUTO])
    for mode in (cks.SORT_SINGLE, cks.SORT_PREFIX):
        assert np.array_equal(res[mode]["mask"], res[cks.SORT_PREFIX_AUTO]["mask"])
        assert np.array_equal(u32(res[mode]["perm"]), u32(res[cks.SORT_PREFIX_AUTO]["perm"]))
        assert np.array_equal(u16(res[mode]["dbit"]), u16(res[cks.SORT_PREFIX_AUTO]["dbit"]))
        assert np.array_equal(u32(res[mode]["packed"]), u32(res[cks.SORT_PREFIX_AUTO]["packed"]))


def test_full_key_build():
    # NEXT-2: the full-key pipeline (M = every key bit) reaches the same exact D and order
    keys = cksgen.config(3, n=40_000)
    try:
        cks.set_sort_mode(cks.SORT_SINGLE)
        r = cks.build(dev(keys), prior_mask=np.full(keys.shape[1], 0xFF, np.uint8))
    finally:
        cks.set_sort_mode(cks.SORT_PREFIX_AUTO)
    assert r["sort_bits"] == 8 * keys.shape[1]
    check_build(keys, r)


def test_sort_mode_rejects():
    with pytest.raises(cks.CksError):
        cks.set_sort_mode(7)


# ---- NEXT-3: the paper's index tree format --------------------------------------------------

@pytest.mark.parametrize("cfg,n,pk,fill", [(1, 13, 32, 0.9), (5, 4097, 32, 0.9), (3, 100_003, 32, 0.9),
                                           (4, 60_000, 17, 0.9), (2, 77_777, 8, 1.0), (1, None, 32, 0.9)])
def test_paper_tree_vs_oracle(cfg, n, pk, fill):
    keys = cksgen.config(cfg, n=n)
    d = dev(keys)
    b = cks.Builder(keys.shape[0], keys.shape[1], d.device)
    b(d)
    nodes = cks.paper_tree(d, b.perm[:keys.shape[0]], b.dbit[:keys.shape[0]], pk_bits=pk, fill=fill)
    ref = oracle.paper_tree(keys, u32(b.perm)[:keys.shape[0]], u16(b.dbit)[:keys.shape[0]], pk=pk, fill=fill)
    assert nodes.shape[0] == sum(ref["levels"])
    assert np.array_equal(nodes.cpu().numpy(), ref["nodes"])


@pytest.mark.parametrize("cfg,n", [(1, 30_001), (3, 80_000), (5, 90_001), (2, 50_000)])
def test_ds_metadata_first_build_and_rebuild(cfg, n):
    # DS-metadata recompute: the variant bitmap V and the reference key come out of
    # the first build (from its superset pass) and of a rebuild (one more pass over the keys)
    keys = cksgen.config(cfg, n=n)
    d = dev(keys)
    V = oracle.variant_bitmap(keys)
    r = cks.build(d, ds_metadata=True)
    assert np.array_equal(r["variant"], V) and np.array_equal(r["ref_key"], keys[0])
    r2 = cks.build(d, prior_mask=r["mask"], ds_metadata=True)
    assert np.array_equal(r2["variant"], V) and np.array_equal(r2["ref_key"], keys[0])
    check_build(keys, r2)
    # D is a subset of V: every distinction bit varies
    assert positions(r["mask"]) <= positions(V)


@pytest.mark.parametrize("cfg,n,pk,fill", [(1, 13, 32, 0.9), (5, 40_963, 32, 0.9), (3, 100_003, 32, 0.9),
                                           (4, 60_000, 17, 0.9), (2, 77_777, 8, 1.0), (1, None, 32, 0.9),
                                           (5, 1, 32, 0.9), (3, 5000, 1, 0.5)])
def test_paper_tree_ds_sources_vs_oracle(cfg, n, pk, fill):
    # NEXT-3 partial keys from the paper's sources: A = the sorted compressed key
    # (P_D from the build), B = the reference key for invariant bits, C(b) = the key row only
    # for variant bits outside D. The node images must equal the oracle's (bits from the rows)
    keys = cksgen.config(cfg, n=n)
    N, B = keys.shape
    d = dev(keys)
    r = cks.build(d, ds_metadata=True)
    perm, dbit = r["perm"], r["dbit"]
    nodes = cks.paper_tree_ds(d, N, B, perm, dbit, r["packed"], N, r["mask"], r["variant"], r["ref_key"], pk, fill)
    ref = oracle.paper_tree(keys, u32(perm), u16(dbit), pk=pk, fill=fill)
    assert np.array_equal(nodes.cpu().numpy(), ref["nodes"])
    # with every variant bit in the planes' mask no row is read: keys may be NULL
    if positions(r["variant"]) <= positions(r["mask"]):
        nodes2 = cks.paper_tree_ds(None, N, B, perm, dbit, r["packed"], N, r["mask"], r["variant"], r["ref_key"],
                                   pk, fill)
        assert np.array_equal(nodes2.cpu().numpy(), ref["nodes"])
    elif N:
        with pytest.raises(cks.CksError):
            cks.paper_tree_ds(None, N, B, perm, dbit, r["packed"], N, r["mask"], r["variant"], r["ref_key"], pk, fill)


@pytest.mark.parametrize("src", [cks.PTREE_AUTO, cks.PTREE_ROWS, cks.PTREE_DS, cks.PTREE_CARRY, cks.PTREE_DECODE])
@pytest.mark.parametrize("cfg,n,pk,fill,ds", [(5, 120_001, 32, 0.9, False), (5, 70_001, 17, 1.0, True),
                                              (3, 90_000, 32, 0.9, True), (4, 50_000, 32, 0.9, False),
                                              (1, None, 24, 0.9, False), (2, 40_000, 32, 0.9, True)])
def test_build_fused_paper_tree(cfg, n, pk, fill, ds, src):
    # cks_build with ptree_nodes: the paper-format tree from the same call, from each of the
    # paper's partial-key sources. With CARRY on cfg5 the variant bits outside the sort mask that
    # partial keys need ride through the sort as one more plane (C(a)); the build's own outputs
    # must not change
    keys = cksgen.config(cfg, n=n)
    if src == cks.PTREE_DECODE and cfg in (1, 3, 4):
        # DECODE reads the sorted P_{D+}, which these builds do not keep (P_M by row id)
        with pytest.raises(cks.CksError):
            cks.build(dev(keys), paper_tree_pk=pk, paper_tree_fill=fill, paper_tree_source=src)
        return
    r = cks.build(dev(keys), paper_tree_pk=pk, paper_tree_fill=fill, ds_metadata=ds, paper_tree_source=src)
    check_build(keys, r)
    ref = oracle.paper_tree(keys, u32(r["perm"]), u16(r["dbit"]), pk=pk, fill=fill)
    assert np.array_equal(r["paper_tree"].cpu().numpy(), ref["nodes"])


@pytest.mark.parametrize("src", [cks.PTREE_DECODE, cks.PTREE_ROWS, cks.PTREE_DS])
@pytest.mark.parametrize("cfg", [5, 2])
@pytest.mark.parametrize("n,fill,pk", [(1, 0.9, 32), (2, 0.9, 32), (13, 0.9, 32), (14, 1.0, 32), (15, 1.0, 32),
                                       (25, 0.9, 5), (43, 0.23, 32), (1000, 0.23, 7), (12 * 8 * 8 + 1, 0.9, 32),
                                       (12 * 8 * 8 * 8 + 11, 0.9, 31)])
def test_fused_paper_tree_shapes(cfg, n, fill, pk, src):
    # the tree's edge shapes through the fused build: one leaf (no inner level), a last leaf of
    # one key (its unused slots zeroed by one thread), the smallest fill (3 per leaf, 2 per inner
    # node), a root over a single child, and the per-level summaries on trees 2-4 levels high
    keys = cksgen.config(cfg, n=n)
    r = cks.build(dev(keys), paper_tree_pk=pk, paper_tree_fill=fill, paper_tree_source=src, ds_metadata=True)
    check_build(keys, r)
    ref = oracle.paper_tree(keys, u32(r["perm"]), u16(r["dbit"]), pk=pk, fill=fill)
    assert r["paper_tree"].shape[0] == sum(ref["levels"])
    assert np.array_equal(r["paper_tree"].cpu().numpy(), ref["nodes"])


@pytest.mark.parametrize("T", [24, 40, 64])
def test_fused_paper_tree_forced_round0(T):
    # the appended plane through every round-0 width (T < 32 leaves 4 remaining words: the
    # compaction path; T = 40 / 64 the register finisher with 4 planes)
    keys = cksgen.config(5, n=66_000)
    cks.set_round0_bits(T)
    try:
        r = cks.build(dev(keys), paper_tree_pk=32, paper_tree_source=cks.PTREE_CARRY)
    finally:
        cks.set_round0_bits(0)
    check_build(keys, r)
    ref = oracle.paper_tree(keys, u32(r["perm"]), u16(r["dbit"]), pk=32, fill=0.9)
    assert np.array_equal(r["paper_tree"].cpu().numpy(), ref["nodes"])


def test_decode_tree_rejects_prior_mask():
    # with a prior mask the sort mask need not separate every byte value: DECODE must refuse
    # unless the D+ test proved the mask (then it holds D+ and decodes like a first build)
    keys = cksgen.config(5, n=50_000)
    ref = oracle.first_build(keys)
    with pytest.raises(cks.CksError):
        cks.build(dev(keys), prior_mask=ref["mask"], paper_tree_pk=32, paper_tree_source=cks.PTREE_DECODE)
    r = cks.build(dev(keys), prior_mask=ref["mask"], paper_tree_pk=32)          # AUTO: rows
    t = oracle.paper_tree(keys, u32(r["perm"]), u16(r["dbit"]), pk=32, fill=0.9)
    assert np.array_equal(r["paper_tree"].cpu().numpy(), t["nodes"])
    dplus = oracle.byteocc_superset(keys)
    for src in (cks.PTREE_DECODE, cks.PTREE_AUTO):
        r = cks.build(dev(keys), prior_mask=dplus, paper_tree_pk=32, paper_tree_source=src)
        check_build(keys, r)
        t = oracle.paper_tree(keys, u32(r["perm"]), u16(r["dbit"]), pk=32, fill=0.9)
        assert np.array_equal(r["paper_tree"].cpu().numpy(), t["nodes"])
    cks.set_verify(cks.VERIFY_OFF)                                  # no D+ test: not proven
    try:
        with pytest.raises(cks.CksError):
            cks.build(dev(keys), prior_mask=dplus, paper_tree_pk=32, paper_tree_source=cks.PTREE_DECODE)
    finally:
        cks.set_verify(cks.VERIFY_PRIOR)


def test_decode_tree_with_variant_superset():
    # V contains D+, so a first build sorted by V decodes as well (wider per-byte tables). Bytes
    # from {0x00, 0x03}: D+ = one bit per byte, V = two; 16 bits fit one LSD sort, whose sorted
    # planes the decode reads
    rng = np.random.default_rng(7)
    keys = rng.choice(np.array([0, 3], np.uint8), size=(40_000, 8))
    assert oracle.popcount(oracle.variant_bitmap(keys)) == 16 and oracle.popcount(oracle.byteocc_superset(keys)) == 8
    r = cks.build(dev(keys), superset_kind=cks.SUPERSET_VARIANT, paper_tree_pk=32,
                  paper_tree_source=cks.PTREE_DECODE)
    check_build(keys, r)
    t = oracle.paper_tree(keys, u32(r["perm"]), u16(r["dbit"]), pk=32, fill=0.9)
    assert np.array_equal(r["paper_tree"].cpu().numpy(), t["nodes"])


def test_paper_tree_ds_all_variant_bits_compressed():
    # the packed mask = V (a rebuild sorted by the variant bitmap): partial keys need no rows
    keys = cksgen.config(3, n=60_000)
    N, B = keys.shape
    d = dev(keys)
    V = oracle.variant_bitmap(keys)
    r = cks.build(d, prior_mask=V, ds_metadata=True)
    cks.set_sort_mode(cks.SORT_SINGLE)
    try:
        rv = cks.build(d, prior_mask=V)
    finally:
        cks.set_sort_mode(cks.SORT_PREFIX_AUTO)
    planes = cks.compress(d, V)                                   # P_V in row order ...
    sorted_pv = planes[:, rv["perm"].long()].contiguous()         # ... in sorted order
    nodes = cks.paper_tree_ds(None, N, B, rv["perm"], rv["dbit"], sorted_pv, N, V, V, r["ref_key"], 32, 0.9)
    ref = oracle.paper_tree(keys, u32(rv["perm"]), u16(rv["dbit"]), pk=32, fill=0.9)
    assert np.array_equal(nodes.cpu().numpy(), ref["nodes"])


@pytest.mark.parametrize("seed", [4, 5])
def test_refine_chunk_cta_rounds(seed):
    # 64-byte keys (D+ = 512 bits: more remaining planes than the CTA tier takes), runs of
    # ~1.5k keys tied on the first 80 bits: the long runs fit a CTA, so the next rounds sort
    # them by one CTA each instead of LSD passes (k_ref_cta_chunk)
    keys = hier_keys(60_000, [256] * 64, seed=seed, groups=(40, 7), dup_rows=300)
    r = cks.build(dev(keys))
    check_build(keys, r)


@pytest.mark.parametrize("T", [8, 16, 24, 40, 56, 64])
@pytest.mark.parametrize("m", [72, 92])
def test_refine_forced_round0_width(T, m):
    # P_M of three planes is carried through round 0 and the short ties inside a tile are
    # finished from the sorted planes (k_ref_tile): T < 32 leaves 3 remaining words, T < 64 2,
    # T = 64 1. cks_ctx_set_round0_bits forces T; the result must not depend on it.
    widths = [256] * (m // 8) + ([1 << (m % 8)] if m % 8 else [])
    keys = hier_keys(70_001, widths, seed=T + m, groups=(5, 30), dup_rows=900)
    cks.set_round0_bits(T)
    try:
        r = cks.build(torch.from_numpy(keys).cuda(), tree=False)
    finally:
        cks.set_round0_bits(0)
    assert int(r["sort_bits"]) == m
    check_build(keys, r)


def test_round0_bits_rejects_bad_width():
    for bad in (4, 65, 72, 12):
        with pytest.raises(cks.CksError):
            cks.set_round0_bits(bad)


def test_build_host_batch_pipelined():
    # cks_build_host_batch: three different columns through the double-buffered pipeline
    cols = [cksgen.config(5, n=150_001, seed=s) for s in (11, 12, 13)]
    rs = cks.build_host_batch(cols)
    for keys, r in zip(cols, rs):
        ref = oracle.first_build(keys)
        assert np.array_equal(r["mask"], ref["mask"])
        assert np.array_equal(r["perm"], ref["perm"])
    one = cks.build_host_batch(cols[:1])                       # a batch of one
    assert np.array_equal(one[0]["perm"], rs[0]["perm"])


@pytest.mark.parametrize("B", [5, 13, 24, 100, 255])
def test_build_odd_widths(B):
    # the fused build on key widths off the specialised paths (generic occupancy / compress),
    # past the sample threshold (n >= 65536) and with duplicate rows
    rng = np.random.default_rng(B)
    n = 70_001
    keys = rng.integers(0, 256, (n, B), dtype=np.uint8)
    keys[:, : min(B, 3)] = rng.integers(0, 4, (n, min(B, 3)), dtype=np.uint8)      # shared prefixes
    dup = rng.integers(0, n, 2000)
    keys[rng.integers(0, n, 2000)] = keys[dup]
    check_build(keys, cks.build(dev(keys)))


def test_build_unaligned_keys():
    # a key column that starts 3 bytes into its buffer (no 16-byte vector paths)
    keys = cksgen.config(3, n=50_001)
    buf = torch.zeros(keys.size + 3, dtype=torch.uint8, device="cuda")
    view = buf[3:].view(keys.shape[0], keys.shape[1])
    view.copy_(dev(keys))
    check_build(keys, cks.build(view))


def test_checked_library_cases():
    # the bounds-checked build (device asserts at computed-index stores, poisoned scratch,
    # canary bands) over every kernel family; a failed assert or canary is a non-zero exit
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "sanitize_cases.py"), "quick"], cwd=root,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "libcks_checked.so" in r.stdout and "all cases ok" in r.stdout


@pytest.mark.parametrize("T,n,seed", [(24, 50_000, 1), (16, 50_000, 2), (8, 30_000, 3), (24, 3_001, 4)])
def test_packed_from_round0_planes(T, n, seed):
    # a7 without a row gather: P_M of more than three planes (not carried), every D bit among the
    # top 64 P_M bits (keys told apart in their first 12 bytes, letters a-h), and the positions
    # the refinement reordered refreshed in the round-0 planes before the repack. T = 8 / 16
    # ties so many keys that the round-1 list is not saved (the row-gather path instead)
    rng = np.random.default_rng(seed)
    keys = np.empty((n, 32), np.uint8)
    keys[:, :12] = rng.integers(0x61, 0x69, size=(n, 12), dtype=np.uint8)
    keys[:, 12:] = rng.integers(0, 256, size=(n, 20), dtype=np.uint8)
    cks.set_round0_bits(T)
    try:
        r = cks.build(dev(keys))
    finally:
        cks.set_round0_bits(0)
    check_build(keys, r)


def test_abi_argument_errors():
    # the header's error contract at the boundary: n >= 2^32 -> CKS_ERANGE (row ids are u32),
    # key_bytes outside [1, 512] or a NULL key pointer with n > 0 -> CKS_EINVAL; nothing is
    # launched (the pointer below addresses one row only)
    import ctypes
    L, c = cks._context(0)
    keys = torch.zeros((1, 16), dtype=torch.uint8, device="cuda")
    mask = np.zeros(512, np.uint8)
    pc = ctypes.c_uint32()
    p = ctypes.c_void_p(keys.data_ptr())
    assert L.cks_superset_mask(c, p, 1 << 32, 16, cks.SUPERSET_BYTEOCC, mask.ctypes.data, ctypes.byref(pc)) == cks.CKS_ERANGE
    assert L.cks_superset_mask(c, p, 1, 0, cks.SUPERSET_BYTEOCC, mask.ctypes.data, ctypes.byref(pc)) == cks.CKS_EINVAL
    assert L.cks_superset_mask(c, p, 1, 513, cks.SUPERSET_BYTEOCC, mask.ctypes.data, ctypes.byref(pc)) == cks.CKS_EINVAL
    assert L.cks_superset_mask(c, None, 5, 16, cks.SUPERSET_BYTEOCC, mask.ctypes.data, ctypes.byref(pc)) == cks.CKS_EINVAL
    assert L.cks_superset_mask(c, None, 0, 16, cks.SUPERSET_BYTEOCC, mask.ctypes.data, ctypes.byref(pc)) == cks.CKS_OK
    torch.cuda.synchronize()
    # the context stays usable after the rejected calls
    k = cksgen.config(1, n=1000)
    check_build(k, cks.build(dev(k)))


def test_prior_mask_proven_by_occupancy():
    # CKS_VERIFY_PRIOR first tries the sufficient test D+(new keys) inside the prior mask (the
    # compress marks the occupancy; one finalize launch more than a rebuild without the check);
    # only when it fails does the row-gather order check run, and a mask that failed is
    # remembered (no occupancy marking next time)
    def launches_of(fn):
        torch.cuda.synchronize()
        a = cks.launches()
        r = fn()
        torch.cuda.synchronize()
        return r, cks.launches() - a

    def rebuild(d, m, mode):
        cks.set_verify(mode)
        try:
            return launches_of(lambda: cks.build(d, prior_mask=m))
        finally:
            cks.set_verify(cks.VERIFY_PRIOR)

    # a prior mask holding D+ (at cfg5's full size the exact D is D+ itself; here, 60 k keys,
    # the exact D is narrower) proves itself: no order check
    keys = cksgen.config(5, n=60_000)
    ref = oracle.first_build(keys)
    d = dev(keys)
    dplus = oracle.byteocc_superset(keys)
    r_off, l_off = rebuild(d, dplus, cks.VERIFY_OFF)
    r_pr, l_pr = rebuild(d, dplus, cks.VERIFY_PRIOR)
    check_build(keys, r_pr)
    assert l_pr == l_off + 1                                     # finalize only, no order check
    # a stale superset of D+ (an extra bit) is proven as well and sorts right
    stale = dplus.copy()
    stale[0] |= 0x80
    r_st, _ = rebuild(d, stale, cks.VERIFY_PRIOR)
    check_build(keys, r_st)
    assert r_st["sort_bits"] == oracle.popcount(stale)             # the paper's rebuild: by the given mask
    # the exact D of 60 k keys is inside D+ but not equal: the test fails, the order check runs;
    # the second rebuild with the same mask skips the occupancy pass
    _, l_off = rebuild(d, ref["mask"], cks.VERIFY_OFF)
    r1, l1 = rebuild(d, ref["mask"], cks.VERIFY_PRIOR)
    r2, l2 = rebuild(d, ref["mask"], cks.VERIFY_PRIOR)
    check_build(keys, r1)
    check_build(keys, r2)
    assert l1 > l2 > l_off and l1 - l2 == 1


@pytest.mark.parametrize("cfg,n", [(1, None), (3, 30_001), (4, 20_003), (2, 50_000)])
def test_decode_tree_single_sort_plane_counts(cfg, n):
    # the decode source over every plane count: one LSD sort keeps P_{D+} sorted whatever its
    # width -- cfg2 1 plane, cfg1 4 (the register path's largest), cfg3 7 and cfg4 12 (the
    # generic path reading the planes from memory)
    keys = cksgen.config(cfg, n=n)
    cks.set_sort_mode(cks.SORT_SINGLE)
    try:
        r = cks.build(dev(keys), paper_tree_pk=32, paper_tree_source=cks.PTREE_DECODE)
    finally:
        cks.set_sort_mode(cks.SORT_PREFIX_AUTO)
    check_build(keys, r)
    t = oracle.paper_tree(keys, u32(r["perm"]), u16(r["dbit"]), pk=32, fill=0.9)
    assert np.array_equal(r["paper_tree"].cpu().numpy(), t["nodes"])


@pytest.mark.parametrize("values", [2, 8])
def test_speculative_mask_retry(values):
    # first builds of >= 2^20 keys take the mask from a strided row sample and let the compress
    # mark the occupancy; when the sample misses a byte value that adds a D+ bit, the build is
    # redone by the full D+. Here one unsampled row carries a value no other row has at byte 3
    # (2 values per byte: one LSD sort; 8: the sort by distinguishing prefixes)
    n = 2_000_003
    rng = np.random.default_rng(11)
    keys = rng.integers(0, values, size=(n, 32), dtype=np.uint8)
    keys[:, 0] = rng.integers(0, 256, size=n, dtype=np.uint8)
    keys[777_777, 3] = 0x80                                       # not on the sample's stride
    d = dev(keys)
    torch.cuda.synchronize()
    a = cks.launches()
    s0 = cks.speculation_stats()
    r = cks.build(d)
    torch.cuda.synchronize()
    l_retry = cks.launches() - a
    s1 = cks.speculation_stats()
    assert (s1[0] - s0[0], s1[1] - s0[1]) == (1, 1)               # speculated, rebuilt once
    check_build(keys, r)
    assert r["sort_bits"] == oracle.popcount(oracle.byteocc_superset(keys))   # sorted by the full D+
    assert np.array_equal(r["sort_mask"], oracle.byteocc_superset(keys))
    keys[777_777, 3] = 0x01                                       # the sample now sees every value
    d = dev(keys)
    torch.cuda.synchronize()
    a = cks.launches()
    r = cks.build(d)
    torch.cuda.synchronize()
    l_plain = cks.launches() - a
    s2 = cks.speculation_stats()
    assert (s2[0] - s1[0], s2[1] - s1[1]) == (1, 0)
    check_build(keys, r)
    assert l_retry > l_plain                                      # the first build ran twice
    cks.set_speculative_mask(False)                               # its own superset pass instead
    try:
        check_build(keys, cks.build(d))
        assert cks.speculation_stats() == s2
    finally:
        cks.set_speculative_mask(True)


@pytest.mark.parametrize("cfg,src", [(5, cks.PTREE_AUTO), (5, cks.PTREE_DS), (3, cks.PTREE_ROWS), (2, cks.PTREE_DECODE)])
def test_speculative_build_with_tree_and_metadata(cfg, src):
    # the speculative first build (>= 2^20 keys) with the DS-metadata and the paper tree: V and
    # the decode tables come from the occupancy the compress marked
    keys = cksgen.config(cfg, n=1_200_007)
    r = cks.build(dev(keys), paper_tree_pk=32, paper_tree_source=src, ds_metadata=True)
    check_build(keys, r)
    assert np.array_equal(r["variant"], oracle.variant_bitmap(keys)) and np.array_equal(r["ref_key"], keys[0])
    t = oracle.paper_tree(keys, u32(r["perm"]), u16(r["dbit"]), pk=32, fill=0.9)
    assert np.array_equal(r["paper_tree"].cpu().numpy(), t["nodes"])


def test_speculative_build_through_every_entry():
    # the speculative first build behind the north-star call cks_distinction_mask, with the
    # order check on every build, and with keys that are not 16-byte aligned (no speculation)
    keys = cksgen.config(3, n=1_100_003)
    d = dev(keys)
    ref = oracle.first_build(keys)
    mask, perm = cks.distinction_mask(d)
    assert np.array_equal(mask, ref["mask"]) and np.array_equal(u32(perm), ref["perm"])
    cks.set_verify(cks.VERIFY_ALWAYS)
    try:
        check_build(keys, cks.build(d))
    finally:
        cks.set_verify(cks.VERIFY_PRIOR)
    raw = torch.zeros(keys.size + 8, dtype=torch.uint8, device="cuda")
    view = raw[8:].view(keys.shape)                                # 8-byte aligned only
    view.copy_(d)
    check_build(keys, cks.build(view))

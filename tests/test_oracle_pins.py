"""Pins for the CPU oracle (oracle/): values the paper prints, closed forms,
invariants (Lemma 1, Theorems 1 and 2), special cases that reduce to textbook or
library routines, and brute force on tiny inputs. None of these re-types the
oracle's own loops: each compares it with something the paper or mathematics
fixes independently. CPU only."""
import itertools

import numpy as np
import pytest

import cksgen
import oracle
from conftest import load_bit_rows, load_hex_keys, mask_from, positions


# ---- independent helpers (integer arithmetic, not the oracle's bit loops) ----

def int_dbit(a: bytes, b: bytes):
    """Most significant differing bit via integer XOR and bit_length (closed form)."""
    x = int.from_bytes(a, "big") ^ int.from_bytes(b, "big")
    return None if x == 0 else 8 * len(a) - x.bit_length()


def py_sorted_perm(keys, rid=None):
    n = keys.shape[0]
    rid = np.arange(n, dtype=np.uint32) if rid is None else rid
    rows = sorted(range(n), key=lambda i: (bytes(keys[i]), int(rid[i])))
    return np.array([rid[i] for i in rows], dtype=np.uint32)


def planes_to_ints(planes):
    np_, n = planes.shape
    return [sum(int(planes[q, i]) << (32 * q) for q in range(np_)) for i in range(n)]


# ---- Fig. 2 worked example (Sec. 3.1) --------------------------------

FIG2 = load_hex_keys("fig2_keys.txt")


def bits12(p):
    return {x for x in p if x < 12}


def test_fig2_distinction_positions():
    # P:218 "bit positions 1, 2, 5 and 7 are distinction bit positions"
    perm = oracle.sort_keys(FIG2)
    assert list(perm) == list(range(6))                      # rows are key_0 < ... < key_5
    dbit, mask = oracle.adjacent_dbits(FIG2, perm)
    assert positions(mask) == {1, 2, 5, 7}
    # D_1 = D_4 = 5, D_2 = 1; D_3 = 7
    assert dbit[1] == 5 and dbit[4] == 5 and dbit[2] == 1 and dbit[3] == 7
    assert dbit[0] == oracle.NONE16
    # Theorem 1: all pairs give the same set
    assert positions(oracle.dbits_all_pairs(FIG2)) == {1, 2, 5, 7}


def test_fig2_lemma1_examples():
    # D-bit(key_1, key_3) = 1 and D-bit(key_0, key_2) = 1
    assert oracle.dbit_pair(FIG2[1], FIG2[3]) == 1
    assert oracle.dbit_pair(FIG2[0], FIG2[2]) == 1


def test_fig2_variant_and_invariant():
    # invariant {0,3,4,8,9,10}, variant {1,2,5,6,7,11}
    v = bits12(positions(oracle.variant_bitmap(FIG2)))
    assert v == {1, 2, 5, 6, 7, 11}
    assert set(range(12)) - v == {0, 3, 4, 8, 9, 10}
    # 6 and 11 variant but not distinction; every distinction bit is variant
    assert {6, 11} <= v and not ({6, 11} & {1, 2, 5, 7})


def test_fig2_deletion_narrative():
    # delete key_3 -> 7 not a distinction position, still variant
    k = np.delete(FIG2, 3, axis=0)
    _, d = oracle.adjacent_dbits(k, oracle.sort_keys(k))
    assert positions(d) == {1, 2, 5}
    assert 7 in positions(oracle.variant_bitmap(k))
    # ... also delete key_0: distinction positions unchanged, 7 becomes invariant
    k2 = np.delete(k, 0, axis=0)
    _, d2 = oracle.adjacent_dbits(k2, oracle.sort_keys(k2))
    assert positions(d2) == {1, 2, 5}
    assert 7 not in positions(oracle.variant_bitmap(k2))


def test_fig2_compressed_keys_and_order():
    # Fig. 2(b) / Theorem 2: compressed keys on positions {1,2,5,7}
    mask = mask_from({1, 2, 5, 7}, 2)
    planes = oracle.compress(FIG2, mask)
    assert planes.shape == (1, 6)
    assert list(planes[0]) == [0b0001, 0b0010, 0b1000, 0b1001, 0b1010, 0b1100]
    assert list(oracle.sort_packed(planes)) == list(range(6))


def test_fig2_doffset():
    # P:479 D-offset[i] = position of the (i+1)-st 1
    assert list(oracle.doffset(mask_from({1, 2, 5, 7}, 2))) == [1, 2, 5, 7]
    assert oracle.doffset(np.zeros(2, np.uint8)).size == 0


# ---- Remark 1 -------------------------------------------------

def test_remark1_not_minimal():
    keys = load_hex_keys("remark1_keys.txt")
    _, d = oracle.adjacent_dbits(keys, oracle.sort_keys(keys))
    assert positions(d) == {0, 1, 3}
    order = list(oracle.sort_keys(keys))

    def determines(sub):
        m = mask_from(sub, 1)
        return list(oracle.sort_packed(oracle.compress(keys, m))) == order and \
            len(set(planes_to_ints(oracle.compress(keys, m)))) == 4
    minimal = [set(s) for r in range(0, 5) for s in itertools.combinations(range(4), r) if determines(s)]
    best = min(len(s) for s in minimal)
    assert best == 2 and [s for s in minimal if len(s) == 2] == [{2, 3}]
    assert determines({0, 1, 3})


# ---- Table 3 and the Sec. 5.1 segmentation ------------

def test_table3_bitmap_facts():
    m = load_bit_rows("table3_indbtab_dbitmap.txt")
    assert m.size == 35                                   # INDBTAB keys are 35 B (Table 2)
    assert oracle.popcount(m) == 56
    last_byte = max(p // 8 for p in positions(m)) + 1     # 1-based byte number
    assert last_byte == 22                                # P:603 "in the 22nd byte"
    assert (oracle.popcount(m) + 7) // 8 == 7             # "stored in 7 bytes"
    st, bits = oracle.pext_segments(m)
    assert list(st + 1) == [3, 11, 19] and list(bits) == [15, 26, 15]
    assert sum(bits) == 56


def test_pext_pipeline_equals_bit_loop():
    # Sec. 5.1 PEXT pipeline vs the plain concatenation of P:223
    rng = np.random.default_rng(7)
    for B in (1, 3, 8, 13, 35, 64):
        keys = rng.integers(0, 256, size=(300, B), dtype=np.uint8)
        for density in (0.05, 0.3, 0.9):
            mask = np.packbits(rng.random(8 * B) < density)
            a = oracle.compress(keys, mask)
            b = oracle.compress(keys, mask, pext=True)
            assert np.array_equal(a, b)
    t3 = load_bit_rows("table3_indbtab_dbitmap.txt")
    keys = rng.integers(0, 256, size=(500, 35), dtype=np.uint8)
    assert np.array_equal(oracle.compress(keys, t3), oracle.compress(keys, t3, pext=True))


# ---- D-bit, Lemma 1, Theorem 1 --------------------------------------------------

def test_dbit_pair_closed_form():
    rng = np.random.default_rng(1)
    for B in (1, 2, 5, 16, 33):
        for _ in range(300):
            a = rng.integers(0, 256, B, dtype=np.uint8)
            b = a.copy()
            j = rng.integers(0, B)
            b[j:] = rng.integers(0, 256, B - j, dtype=np.uint8)
            d = oracle.dbit_pair(a, b)
            e = int_dbit(bytes(a), bytes(b))
            assert (d == -1 and e is None) or d == e


@pytest.mark.parametrize("seed", range(6))
def test_lemma1_and_theorem1_bruteforce(seed):
    rng = np.random.default_rng(seed)
    B = int(rng.integers(1, 6))
    n = int(rng.integers(2, 65))
    keys = rng.integers(0, 256, size=(n, B), dtype=np.uint8)
    keys &= rng.integers(0, 256, size=B, dtype=np.uint8)          # shared zero bits
    keys = np.unique(keys, axis=0)                                 # Lemma 1 is stated for distinct keys
    rng.shuffle(keys)
    perm = oracle.sort_keys(keys)
    s = keys[perm]
    dbit, d = oracle.adjacent_dbits(keys, perm)
    for i in range(len(s)):
        for j in range(i + 1, len(s)):
            assert int_dbit(bytes(s[i]), bytes(s[j])) == int(dbit[i + 1:j + 1].min())   # Lemma 1
    assert positions(d) == positions(oracle.dbits_all_pairs(keys))                      # Theorem 1


def test_sort_keys_matches_library_sort():
    rng = np.random.default_rng(3)
    keys = cksgen.uniform(2000, 5, seed=11, dup_ppm=100000)
    assert np.array_equal(oracle.sort_keys(keys), py_sorted_perm(keys))
    rid = rng.permutation(2000).astype(np.uint32)
    assert np.array_equal(oracle.sort_keys(keys, rid=rid), py_sorted_perm(keys, rid))
    assert np.array_equal(oracle.sort_keys(keys, threads=4), py_sorted_perm(keys))


@pytest.mark.slow
def test_theorem1_cfg1_all_pairs():
    # cfg1 at full size: all 2.1e9 pairs == sorted adjacency
    keys = cksgen.config(1)
    _, d = oracle.adjacent_dbits(keys, oracle.sort_keys(keys, threads=oracle.threads_default()))
    assert positions(d) == positions(oracle.dbits_all_pairs(keys))


# ---- special cases with closed forms ----------------------------------------------

def test_special_cases():
    # all 2^16 distinct 2-byte keys -> every bit is a distinction bit
    k = cksgen.consecutive(1 << 16, 2, shuffle_seed=5)
    _, d = oracle.adjacent_dbits(k, oracle.sort_keys(k))
    assert positions(d) == set(range(16))
    # consecutive integers 0..2^k-1 -> the low k bits
    for kk in (1, 5, 9):
        k = cksgen.consecutive(1 << kk, 4, shuffle_seed=kk)
        _, d = oracle.adjacent_dbits(k, oracle.sort_keys(k))
        assert positions(d) == set(range(32 - kk, 32))
    # all equal / n <= 1 -> empty
    for n in (0, 1, 7):
        k = cksgen.all_equal(n, 9, seed=2)
        _, d = oracle.adjacent_dbits(k, oracle.sort_keys(k))
        assert positions(d) == set()
        assert positions(oracle.byteocc_superset(k)) == set()
        assert positions(oracle.variant_bitmap(k)) == set()


def test_identity_mask_compress_is_the_key():
    # all-ones mask over an 8-byte key -> compressed key == key word
    k = cksgen.uniform(500, 8, seed=4)
    planes = oracle.compress(k, np.full(8, 0xFF, np.uint8))
    vals = planes_to_ints(planes)
    assert vals == [int.from_bytes(bytes(r), "big") for r in k]


def test_cfg2_numeric_crosscheck():
    # textbook numeric path: sort the uint64 values, D = {clz64(u_i ^ u_{i+1})}
    k = cksgen.config(2, n=200_000)
    u = np.sort(k.view(">u8").ravel().astype(np.uint64))
    x = u[1:] ^ u[:-1]
    x = x[x != 0]
    exp = {64 - int(v).bit_length() for v in np.unique(x)}
    _, d = oracle.adjacent_dbits(k, oracle.sort_keys(k))
    assert positions(d) == exp
    assert len(exp) <= 23                                # 22 low bits + <= 1 carry position


# ---- supersets: D subset of D+ subset of V, closed forms for D+ -------------------

def test_superset_chain_and_closed_forms():
    for keys in (cksgen.config(1, n=5000), cksgen.config(3, n=20000), cksgen.config(4, n=20000),
                 cksgen.config(5, n=20000), cksgen.config(2, n=20000)):
        _, d = oracle.adjacent_dbits(keys, oracle.sort_keys(keys))
        dp = positions(oracle.byteocc_superset(keys))
        v = positions(oracle.variant_bitmap(keys))
        D = positions(d)
        assert D <= dp <= v
        assert min(v) in D                               # first variant bit separates some pair
    # ACGT bytes: per-byte D+ = {3,5,6} (A 0x41, C 0x43, G 0x47, T 0x54)
    g = cksgen.genome(50_000, seed=9)
    dp = positions(oracle.byteocc_superset(g))
    assert dp == {8 * j + t for j in range(32) for t in (3, 5, 6)}
    # ASCII digits '0'..'9' -> low nibble {4,5,6,7} (cf. Table 3's 00001111 bytes)
    rng = np.random.default_rng(0)
    dig = (0x30 + rng.integers(0, 10, size=(5000, 6))).astype(np.uint8)
    assert positions(oracle.byteocc_superset(dig)) == {8 * j + t for j in range(6) for t in (4, 5, 6, 7)}


# ---- Theorem 2: compressed order == full-key order (with row-id tie-break) ----------

@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_theorem2_on_configs(cfg):
    keys = cksgen.config(cfg, n=30_000)
    permK = oracle.sort_keys(keys)
    assert np.array_equal(permK, py_sorted_perm(keys))
    _, d = oracle.adjacent_dbits(keys, permK)
    rng = np.random.default_rng(cfg)
    B = keys.shape[1]
    masks = [d, oracle.byteocc_superset(keys), oracle.variant_bitmap(keys),
             d | np.packbits(rng.random(8 * B) < 0.2)]          # superset safety
    for m in masks:
        planes = oracle.compress(keys, m)
        assert np.array_equal(oracle.sort_packed(planes), permK)
    # injectivity on distinct keys
    u = np.unique(keys, axis=0)
    pl = oracle.compress(u, d)
    assert len(set(planes_to_ints(pl))) == u.shape[0]


def test_negative_mask_missing_a_distinction_bit():
    # clearing one true D-bit must break Theorem 2's equality for a witness input
    keys = FIG2[::-1].copy()                 # reversed rows: row-id tie-break cannot rescue the order
    permK = oracle.sort_keys(keys)
    for p in (1, 2, 5, 7):
        m = mask_from({1, 2, 5, 7} - {p}, 2)
        assert not np.array_equal(oracle.sort_packed(oracle.compress(keys, m)), permK)


# ---- adjacency on compressed keys ------------------------------------

@pytest.mark.parametrize("cfg", [1, 3, 5])
def test_adjacent_compressed_equals_full_key_dbits(cfg):
    keys = cksgen.config(cfg, n=20_000)
    permK = oracle.sort_keys(keys)
    dfull, d = oracle.adjacent_dbits(keys, permK)
    sup = oracle.byteocc_superset(keys)
    m = oracle.popcount(sup)
    planes = oracle.compress(keys, sup)
    sp = planes[:, oracle.sort_packed(planes)]
    dc, mask = oracle.adjacent_compressed(sp, m, sup)
    assert np.array_equal(dc, dfull)
    assert np.array_equal(mask, d)                      # new D subset of old, here == exact D


# ---- bulk load -----------------------------------------------------------

@pytest.mark.parametrize("n,fanout,fill", [(1, 64, 1.0), (64, 64, 1.0), (65, 64, 1.0),
                                           (20_000, 64, 1.0), (5000, 14, 0.9), (3000, 9, 0.9)])
def test_bulkload_structure(n, fanout, fill):
    keys = cksgen.config(3, n=n)
    perm = oracle.sort_keys(keys)
    dbit, _ = oracle.adjacent_dbits(keys, perm)
    t = oracle.bulkload(perm, dbit, keys, fanout, fill)
    per = int(np.floor(fanout * fill))
    # closed forms: leaf count ceil(n/per); height = levels until one node
    assert t["level_nodes"][0] == -(-n // per)
    h, c = 1, -(-n // per)
    while c > 1:
        c = -(-c // per)
        h += 1
    assert t["height"] == h and t["level_nodes"][-1] == 1
    L0 = int(t["level_nodes"][0])
    leaf_rids = t["entry_rid"][:L0, :per].ravel()
    assert np.array_equal(leaf_rids[leaf_rids != 0xFFFFFFFF], perm)      # leaf scan == perm
    assert t["node_cnt"][:L0].sum() == n
    # inner D-bits: the direct formula == range-min of D_k (Lemma 1)
    off, span = L0, per
    for lvl in range(1, t["height"]):
        nodes = int(t["level_nodes"][lvl])
        ent = t["entry_rid"][off:off + nodes, :per].ravel()
        edb = t["entry_dbit"][off:off + nodes, :per].ravel()
        cnt = int(t["node_cnt"][off:off + nodes].sum())
        for x in range(1, cnt):
            lo, hi = x * span, min((x + 1) * span, n) - 1   # (prev entry's highest, this highest]
            expect = int(dbit[lo:hi + 1].min())
            assert edb[x] == expect
            assert ent[x] == perm[hi]
        assert edb[0] == oracle.NONE16
        off += nodes
        span *= per


# ---- NEXT-3: the paper's index tree format (Sec. 4.2, Sec. 5.3) ---------------------------

def le(nd, off, size):
    return int.from_bytes(bytes(nd[off:off + size]), "little")


def test_paper_tree_fig2_partial_key():
    # "the partial key of key_1 when pk = 4 is 1010, because D_1 = 5"
    perm = np.arange(6, dtype=np.uint32)                          # FIG2 rows are in sorted order
    dbit, _ = oracle.adjacent_dbits(FIG2, perm)
    t = oracle.paper_tree(FIG2, perm, dbit, pk=4, fill=0.9)
    assert t["height"] == 1 and t["leaf_per"] == 12 and t["inner_per"] == 8   # floor(14*.9), floor(9*.9)
    leaf = t["nodes"][0]
    assert le(leaf, 0, 2) == 6 and le(leaf, 2, 2) == 0 and le(leaf, 8, 8) == 5
    assert le(leaf, 24, 8) == (1 << 64) - 1                       # no next leaf
    e1 = leaf[32 + 16:32 + 32]
    assert le(e1, 0, 4) >> 28 == 0b1010
    assert le(e1, 4, 2) == 5 and le(e1, 6, 2) == 2 and le(e1, 8, 8) == 1


def ref_partial_key(key: bytes, d, pk):
    """pk bits after position d (reading C14) via big-integer shifts."""
    v = int.from_bytes(key, "big")
    nb = 8 * len(key)
    start = 0 if d is None else d + 1
    out = 0
    for j in range(pk):
        p = start + j
        out = (out << 1) | ((v >> (nb - 1 - p)) & 1 if p < nb else 0)
    return out << (32 - pk)


@pytest.mark.parametrize("n,fill,pk", [(1, 0.9, 32), (12, 0.9, 32), (13, 0.9, 16), (1000, 0.9, 32),
                                      (20_000, 1.0, 24)])
def test_paper_tree_structure(n, fill, pk):
    keys = cksgen.config(3, n=n) if n > 1 else cksgen.uniform(1, 32, seed=3)
    perm = oracle.sort_keys(keys)
    dbit, _ = oracle.adjacent_dbits(keys, perm)
    t = oracle.paper_tree(keys, perm, dbit, pk=pk, fill=fill)
    lp, ip = t["leaf_per"], t["inner_per"]
    # node counts: ceil(n / per) per level
    lv, c = [-(-n // lp)], -(-n // lp)
    while c > 1:
        c = -(-c // ip)
        lv.append(c)
    assert t["levels"] == lv
    nodes = t["nodes"]
    # leaves in order hold the sorted record ids; headers point at the highest key; next chain
    rids = [le(nodes[j], 32 + 16 * e + 8, 8) for j in range(lv[0]) for e in range(le(nodes[j], 0, 2))]
    assert rids == [int(x) for x in perm]
    for j in range(lv[0]):
        cnt = le(nodes[j], 0, 2)
        assert le(nodes[j], 8, 8) == le(nodes[j], 32 + 16 * (cnt - 1) + 8, 8)
        assert le(nodes[j], 24, 8) == (j + 1 if j + 1 < lv[0] else (1 << 64) - 1)
    # partial keys against a big-integer re-derivation on sampled entries
    rng = np.random.default_rng(n)
    for k in rng.choice(n, min(n, 200), replace=False):
        j, e = divmod(int(k), lp)
        ent = nodes[j][32 + 16 * e: 48 + 16 * e]
        d = None if dbit[k] == 0xFFFF else int(dbit[k])
        assert le(ent, 0, 4) == ref_partial_key(bytes(keys[perm[k]]), d, pk)
    # inner entries: child index, highest key, and the D-bit against the previous entry's
    # highest key equals the minimum D_k over the child's keys (Lemma 1)
    off, below, cover = lv[0], 0, lp
    for l in range(1, len(lv)):
        for j in range(lv[l]):
            nd = nodes[off + j]
            assert le(nd, 2, 2) == l
            for e in range(le(nd, 0, 2)):
                ch = j * ip + e
                ent = nd[24 + 24 * e: 48 + 24 * e]
                hi = min((ch + 1) * cover, n) - 1
                assert le(ent, 8, 8) == below + ch and le(ent, 16, 8) == perm[hi]
                want = 0xFFFF if ch == 0 else int(dbit[ch * cover: hi + 1].min())
                assert le(ent, 4, 2) == want
        below, off, cover = off, off + lv[l], cover * ip


# ---- P:502 block-parallel construction (orc_bulkload_blocks, NEXT-4's a8) ------------------------

def _subtree_ranges(t, n):
    """(lo, hi) sorted-index range under every node, from the leaf counts upward."""
    lv = [int(x) for x in t["level_nodes"]]
    off = np.cumsum([0] + lv)
    lo = np.zeros(off[-1], np.int64)
    hi = np.zeros(off[-1], np.int64)
    pos = 0
    for j in range(lv[0]):
        c = int(t["node_cnt"][j])
        lo[j], hi[j] = pos, pos + c - 1
        pos += c
    assert pos == n
    for l in range(1, len(lv)):
        for j in range(lv[l]):
            node = off[l] + j
            ch = t["entry_child"][node][: int(t["node_cnt"][node])].astype(np.int64)
            lo[node], hi[node] = lo[ch[0]], hi[ch[-1]]
    return lo, hi


@pytest.mark.parametrize("n,fanout", [(1, 8), (7, 8), (64, 8), (5000, 8), (3001, 16)])
def test_bulkload_blocks_one_block_is_bulkload(n, fanout):
    keys = cksgen.config(3, n=n)
    ref = oracle.first_build(keys)
    a = oracle.bulkload(ref["perm"], ref["dbit"], keys, fanout, 1.0)
    b = oracle.bulkload_blocks(ref["perm"], ref["dbit"], keys, [n], fanout, 1.0)
    assert a["height"] == b["height"]
    for k in ("node_cnt", "entry_rid", "entry_child", "entry_dbit"):
        assert np.array_equal(a[k], b[k])


@pytest.mark.parametrize("blocks", [[64, 64, 64], [512, 512], [64] * 9])
def test_bulkload_blocks_complete_subtrees_equal_global(blocks):
    # blocks of per^k keys: complete subtrees; removing their roots and linking the roots'
    # children gives exactly the global bottom-up bulk load
    n = sum(blocks)
    keys = cksgen.config(5, n=n)
    ref = oracle.first_build(keys)
    a = oracle.bulkload(ref["perm"], ref["dbit"], keys, 8, 1.0)
    b = oracle.bulkload_blocks(ref["perm"], ref["dbit"], keys, blocks, 8, 1.0)
    for k in ("node_cnt", "entry_rid", "entry_child", "entry_dbit"):
        assert np.array_equal(a[k], b[k])


@pytest.mark.parametrize("blocks", [[100, 0, 37, 900], [1, 1, 1], [4000, 10], [333] * 7])
def test_bulkload_blocks_invariants(blocks):
    n = sum(blocks)
    keys = cksgen.config(1, n=n)
    ref = oracle.first_build(keys)
    per = 8
    t = oracle.bulkload_blocks(ref["perm"], ref["dbit"], keys, blocks, per, 1.0)
    lv = [int(x) for x in t["level_nodes"]]
    assert lv[-1] == 1 and all(1 <= c <= per for c in t["node_cnt"])
    leaves = np.concatenate([t["entry_rid"][j][: int(t["node_cnt"][j])] for j in range(lv[0])])
    assert np.array_equal(leaves, ref["perm"])                     # every key once, in order
    nz = [b for b in blocks if b]
    # leaves never straddle a block border (each block is built on its own)
    borders = set(np.cumsum(nz)[:-1].tolist())
    lo, hi = _subtree_ranges(t, n)
    assert all(not (lo[j] < b <= hi[j]) for j in range(lv[0]) for b in borders)
    off = np.cumsum([0] + lv)
    for l in range(1, len(lv)):
        first = True
        for j in range(lv[l]):
            node = off[l] + j
            for e in range(int(t["node_cnt"][node])):
                c = int(t["entry_child"][node][e])
                assert t["entry_rid"][node][e] == ref["perm"][hi[c]]     # highest key of the child
                d = int(t["entry_dbit"][node][e])
                if first:
                    assert d == 0xFFFF
                    first = False
                else:                                                   # Lemma 1 across borders
                    assert d == int(ref["dbit"][lo[c]: hi[c] + 1].min())


def test_generator_frozen():
    # the inputs are frozen: cfg1's column and a prefix of cfg5's hash to the values DESIGN.md
    # section 4 records (a changed generator changes every measured number)
    import hashlib
    assert hashlib.sha256(cksgen.config(1).tobytes()).hexdigest() == \
        "f593de1dd7430bc76b7a93ec24593f8e3a4a6414969583d97fa66f58b191d9fb"
    k5 = cksgen.config(5, n=100_000)
    assert k5.shape == (100_000, 32) and set(np.unique(k5).tolist()) <= {ord(c) for c in "ACGT"}

"""Test infrastructure: the per-shard steps of paper_2009_11543_b200/shard.py on the CPU, from
the oracle (sort, compress, adjacency, bulk load) and plain numpy (occupancy bitsets, lower
bounds, bit repack), so that the sharded orchestration and its collectives can run under
gloo without a GPU. Only tests import this module."""
from types import SimpleNamespace

import numpy as np
import torch

import oracle


def _u32(t: torch.Tensor) -> np.ndarray:
    return np.ascontiguousarray(t.cpu().numpy()).view(np.uint32)


def _i32(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.uint32)).view(np.int32).copy())


def occupancy_np(keys: np.ndarray) -> np.ndarray:
    n, B = keys.shape
    occ = np.zeros((B, 8), np.uint32)
    for j in range(B):
        for v in np.unique(keys[:, j]) if n else []:
            occ[j, v >> 5] |= np.uint32(1 << (int(v) & 31))
    return occ.reshape(-1)


def mask_from_occupancy(occ: np.ndarray, B: int, n_total: int, byteocc: bool = True) -> np.ndarray:
    """D+ (D-bits of the sorted occurring values per byte) or V from an occupancy."""
    occ = occ.reshape(B, 8)
    out = np.zeros(B, np.uint8)
    for j in range(B):
        vals = [w * 32 + b for w in range(8) for b in range(32) if (int(occ[j, w]) >> b) & 1]
        if byteocc:
            for a, c in zip(vals, vals[1:]):
                out[j] |= 0x80 >> (8 - (a ^ c).bit_length())
        elif n_total > 0 and vals:
            o, a = 0, 0xFF
            for v in vals:
                o |= v
                a &= v
            out[j] = o & ~a
    return out


def planes_to_bits(planes: np.ndarray, m: int) -> np.ndarray:
    """[n, m] bit matrix of P (column t = compressed position t, MSB first)."""
    n = planes.shape[1]
    bits = np.zeros((n, m), np.uint8)
    for t in range(m):
        b = m - 1 - t
        bits[:, t] = (planes[b >> 5] >> np.uint32(b & 31)) & 1
    return bits


def bits_to_planes(bits: np.ndarray) -> np.ndarray:
    n, m = bits.shape
    planes = np.zeros((oracle.nplanes(m), n), np.uint32)
    for t in range(m):
        b = m - 1 - t
        planes[b >> 5] |= bits[:, t].astype(np.uint32) << np.uint32(b & 31)
    return planes


class OracleOps:
    """Same interface as shard.CudaOps, on CPU tensors. `all_keys` (the whole column) is only
    for the bulk load, whose oracle computes inner D-bits from the full keys."""

    def __init__(self, all_keys: np.ndarray, superset_byteocc: bool = True):
        self.all_keys = all_keys
        self.byteocc = superset_byteocc

    def occupancy(self, keys):
        return _i32(occupancy_np(keys.cpu().numpy()))

    def occupancy_mask(self, occs, n_total, kind):
        u = np.bitwise_or.reduce(_u32(occs).reshape(occs.shape[0], -1), axis=0)
        return mask_from_occupancy(u, u.size // 8, n_total, self.byteocc)

    def compress(self, keys, mask):
        return _i32(oracle.compress(keys.cpu().numpy(), mask))

    def sort(self, planes, bits, row_ids=None):
        p = _u32(planes).reshape(planes.shape)
        n = p.shape[1]
        rid = None if row_ids is None else _u32(row_ids)
        perm = oracle.sort_packed(p, rid)
        if rid is None:
            order = perm.astype(np.int64)
        else:
            inv = np.argsort(rid, kind="stable")
            order = inv[np.searchsorted(rid[inv], perm)]
        return _i32(perm), _i32(p[:, order] if n else p)

    def rank_sorted(self, sorted_planes, bits, sorted_rid, rid_base, queries):
        p = _u32(sorted_planes).reshape(sorted_planes.shape)
        npl, n = p.shape
        rid = _u32(sorted_rid).astype(np.int64) + rid_base
        q = _u32(queries).reshape(queries.shape)
        out = []
        for row in q:
            lt = np.zeros(n, bool)
            eq = np.ones(n, bool)
            for w in range(npl - 1, -1, -1):
                lt |= eq & (p[w] < row[w])
                eq &= p[w] == row[w]
            lt |= eq & (rid < int(row[npl]))
            out.append(int(lt.sum()))
        return torch.tensor(out, dtype=torch.int64)

    def sort_prefix(self, planes, sort_mask, want_packed=False):
        p = _u32(planes).reshape(planes.shape)
        m = oracle.popcount(sort_mask)
        order = oracle.sort_packed(p)                          # (P, index) order
        dbit, mask = oracle.adjacent_compressed(p[:, order.astype(np.int64)], m, sort_mask)
        return _i32(order), torch.from_numpy(dbit.view(np.int16).copy()), mask, None

    def partition(self, planes, bits, splitters, parts, rid_base):
        p = _u32(planes).reshape(planes.shape)
        npl, n = p.shape
        q = _u32(splitters).reshape(splitters.shape)
        rid = np.arange(n, dtype=np.int64) + rid_base
        dest = np.zeros(n, np.int64)
        for row in q:                                     # count the splitters <= element
            gt = np.zeros(n, bool)
            eq = np.ones(n, bool)
            for w in range(npl - 1, -1, -1):
                gt |= eq & (row[w] > p[w])
                eq &= p[w] == row[w]
            gt |= eq & (int(row[npl]) > rid)
            dest += ~gt
        order = np.argsort(dest, kind="stable")
        return (_i32(p[:, order]), _i32(rid[order].astype(np.uint32)),
                torch.tensor(np.bincount(dest, minlength=parts), dtype=torch.int64))

    def adjacent(self, sorted_planes, bits, sort_mask):
        dbit, mask = oracle.adjacent_compressed(_u32(sorted_planes).reshape(sorted_planes.shape), bits, sort_mask)
        return mask, torch.from_numpy(dbit.view(np.int16).copy())

    def repack(self, planes, in_mask, out_mask):
        m = oracle.popcount(in_mask)
        bits = planes_to_bits(_u32(planes).reshape(planes.shape), m)
        pos = oracle.doffset(in_mask)                         # key bit of each compressed position
        keep = [t for t in range(m) if (int(out_mask[pos[t] >> 3]) >> (7 - (int(pos[t]) & 7))) & 1]
        return _i32(bits_to_planes(bits[:, keep]))

    def bulkload_block(self, perm, dbit, fanout, fill, first_global, levels):
        """Range-minimum bulk load of one block (numpy; the independent check of the result is
        oracle.bulkload_blocks, which takes the D-bits from the keys)."""
        p = _u32(perm)
        d = dbit.cpu().numpy().view(np.uint16).astype(np.int64)
        per = int(fanout * fill)
        lv = oracle.tree_levels(p.size, per)[:levels]
        return self._levels(p, d, lv, fanout, per, first_global, leaves=True)

    def bulkload_top(self, child_rid, child_min, fanout, fill):
        p = _u32(child_rid)
        d = child_min.cpu().numpy().view(np.uint16).astype(np.int64)
        per = int(fanout * fill)
        lv = oracle.tree_levels(p.size, per) if p.size > 1 else []
        t = self._levels(p, d, lv, fanout, per, True, leaves=False)
        t["height"] = len(lv)
        return t

    @staticmethod
    def _levels(p, d, lv, f, per, first_global, leaves):
        n = p.size
        T = int(sum(lv))
        off = np.cumsum([0] + list(lv))
        cnt = np.zeros(max(T, 1), np.uint32)
        rid = np.full(max(T, 1) * f, 0xFFFFFFFF, np.uint32)
        edb = np.full(max(T, 1) * f, 0xFFFF, np.uint16)
        inner0 = lv[0] if leaves and lv else 0
        child = np.full(max(T - inner0, 1) * f, 0xFFFFFFFF, np.uint32)
        rmin, span = d, 1
        for l, nodes in enumerate(lv):
            ents = n if l == 0 else lv[l - 1]
            leaf = leaves and l == 0
            out_min = np.zeros(nodes, np.int64)
            for j in range(nodes):
                xs = range(j * per, min((j + 1) * per, ents))
                node = off[l] + j
                cnt[node] = len(xs)
                for e, x in enumerate(xs):
                    s = node * f + e
                    hi = min((x + 1) * span, n) - 1
                    rid[s] = p[hi]
                    if leaf:
                        edb[s] = d[x]
                    else:
                        edb[s] = 0xFFFF if (x == 0 and first_global) else rmin[x]
                        below = off[l - 1] if (leaves and l > 0) else (0 if l == 0 else off[l - 1])
                        child[(node - inner0) * f + e] = below + x
                out_min[j] = min(rmin[x] for x in xs)
            rmin = out_min
            span *= per
        i32 = lambda a: torch.from_numpy(a.view(np.int32).copy())
        return dict(shape=SimpleNamespace(level_nodes=list(lv), level_offset=list(off[:-1])), node_cnt=i32(cnt),
                    entry_rid=i32(rid), entry_dbit=torch.from_numpy(edb.view(np.int16).copy()), entry_child=i32(child),
                    top_min=torch.from_numpy(rmin.astype(np.uint16).view(np.int16).copy()))


def check_slices(keys, outs, fanout=64, fill=1.0):
    """The ranks' slices, concatenated, against the oracle's single first build."""
    ref = oracle.first_build(keys)
    perm = np.concatenate([o["perm"].cpu().numpy().view(np.uint32) for o in outs])
    dbit = np.concatenate([o["dbit"].cpu().numpy().view(np.uint16) for o in outs])
    assert np.array_equal(perm, ref["perm"])
    assert np.array_equal(dbit, ref["dbit"])
    for o in outs:
        assert np.array_equal(o["mask"], ref["mask"])
    offs = [o["offset"] for o in outs]
    assert offs == list(np.cumsum([0] + [o["perm"].numel() for o in outs])[:-1])
    if ref["m"]:
        packed = np.concatenate([o["packed"].cpu().numpy().view(np.uint32) for o in outs], axis=1)
        assert np.array_equal(packed, ref["planes"][:, ref["perm"]])
    if keys.shape[0] and outs[0].get("tree") is not None:
        from paper_2009_11543_b200 import shard
        got = shard.assemble_tree(outs)
        sizes = [o["perm"].numel() for o in outs]
        exp = oracle.bulkload_blocks(ref["perm"], ref["dbit"], keys, sizes, fanout, fill)
        assert got["height"] == exp["height"]
        assert np.array_equal(got["level_nodes"], exp["level_nodes"])
        for k in ("node_cnt", "entry_rid", "entry_child", "entry_dbit"):
            assert np.array_equal(got[k], exp[k]), k

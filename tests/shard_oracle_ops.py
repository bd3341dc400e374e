"""Test infrastructure: the per-shard steps of paper_2009_11543_b200/shard.py on the CPU, from
the oracle (sort, compress, adjacency, bulk load) and plain numpy (occupancy bitsets, lower
bounds, bit repack), so that the sharded orchestration and its collectives can run under
gloo without a GPU. Only tests import this module."""
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

    def bulkload(self, perm, dbit, fanout, fill):
        return oracle.bulkload(_u32(perm), dbit.cpu().numpy().view(np.uint16), self.all_keys, fanout, fill)


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
    t = outs[0]["tree"]
    if keys.shape[0]:
        exp = oracle.bulkload(ref["perm"], ref["dbit"], keys, fanout, fill)
        T = exp["entry_rid"].size
        rid = t["entry_rid"].cpu().numpy() if torch.is_tensor(t["entry_rid"]) else t["entry_rid"]
        db = t["entry_dbit"].cpu().numpy() if torch.is_tensor(t["entry_dbit"]) else t["entry_dbit"]
        assert np.array_equal(rid.reshape(-1).view(np.uint32)[:T], exp["entry_rid"].ravel())
        assert np.array_equal(db.reshape(-1).view(np.uint16)[:T], exp["entry_dbit"].ravel())

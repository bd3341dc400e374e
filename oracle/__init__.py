"""CPU oracle for the compressed key sort (arXiv 2009.11543) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package. The product path
(``paper_2009_11543_b200``) never imports it and has no CPU fallback.

This is a thin ctypes wrapper over ``oracle.cpp`` (plain C++17, std::sort as the
sort step, bit loops everywhere else). See the citations in oracle.cpp. Every
function here is pinned by ``tests/test_oracle_pins.py`` against facts the paper
states (Fig. 2 / Lemma 1 / Theorem 1 / Remark 1 / Table 3), closed forms and
brute force. Pin status per function is listed in DESIGN.md "Oracle pins";
no function is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None
NONE16 = 0xFFFF


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared",
                               "-o", _SO, src])
    return _SO


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        p, u64, u32, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        L.orc_dbit_pair.argtypes = [p, p, u32]
        L.orc_dbit_pair.restype = i32
        L.orc_dbits_all_pairs.argtypes = [p, u64, u32, p, i32]
        L.orc_sort_keys.argtypes = [p, u64, u32, p, p, i32]
        L.orc_adjacent_dbits.argtypes = [p, u64, u32, p, p, p]
        L.orc_variant_bitmap.argtypes = [p, u64, u32, p]
        L.orc_byteocc_superset.argtypes = [p, u64, u32, p]
        L.orc_doffset.argtypes = [p, u32, p]
        L.orc_doffset.restype = u32
        L.orc_compress.argtypes = [p, u64, u32, p, p]
        L.orc_compress_pext.argtypes = [p, u64, u32, p, p]
        L.orc_pext_segments.argtypes = [p, u32, p, p]
        L.orc_pext_segments.restype = u32
        L.orc_sort_packed.argtypes = [p, u32, u64, p, p, i32]
        L.orc_adjacent_compressed.argtypes = [p, u32, u64, p, u32, p, p]
        L.orc_bulkload.argtypes = [p, p, u64, u32, u32, p, u32, p, p, p, p, p]
        L.orc_bulkload.restype = u32
        L.orc_bulkload_blocks.argtypes = [p, p, u64, p, u32, u32, u32, p, u32, p, p, p, p, p]
        L.orc_bulkload_blocks.restype = u32
        L.orc_paper_tree.argtypes = [p, u64, u32, p, p, u32, u32, u32, p]
        L.orc_paper_tree.restype = u32
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None or a.size == 0 else a.ctypes.data


def _keys(keys) -> np.ndarray:
    k = np.ascontiguousarray(keys, dtype=np.uint8)
    assert k.ndim == 2
    return k


def threads_default() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def dbit_pair(a, b) -> int:
    a = np.ascontiguousarray(a, dtype=np.uint8)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    assert a.shape == b.shape
    return _load().orc_dbit_pair(_ptr(a), _ptr(b), a.size)


def dbits_all_pairs(keys, threads: int | None = None) -> np.ndarray:
    k = _keys(keys)
    n, B = k.shape
    out = np.zeros(B, np.uint8)
    _load().orc_dbits_all_pairs(_ptr(k), n, B, out.ctypes.data, threads or threads_default())
    return out


def sort_keys(keys, rid=None, threads: int = 1) -> np.ndarray:
    k = _keys(keys)
    n, B = k.shape
    perm = np.empty(n, np.uint32)
    r = None if rid is None else np.ascontiguousarray(rid, dtype=np.uint32)
    _load().orc_sort_keys(_ptr(k), n, B, _ptr(r), _ptr(perm), threads)
    return perm


def adjacent_dbits(keys, perm):
    """(dbit[n] uint16, mask[B]) over the sorted order given by perm (row ids = indices)."""
    k = _keys(keys)
    n, B = k.shape
    perm = np.ascontiguousarray(perm, dtype=np.uint32)
    dbit = np.empty(n, np.uint16)
    mask = np.zeros(B, np.uint8)
    _load().orc_adjacent_dbits(_ptr(k), n, B, _ptr(perm), _ptr(dbit), mask.ctypes.data)
    return dbit, mask


def variant_bitmap(keys) -> np.ndarray:
    k = _keys(keys)
    n, B = k.shape
    out = np.zeros(B, np.uint8)
    _load().orc_variant_bitmap(_ptr(k), n, B, out.ctypes.data)
    return out


def byteocc_superset(keys) -> np.ndarray:
    k = _keys(keys)
    n, B = k.shape
    out = np.zeros(B, np.uint8)
    _load().orc_byteocc_superset(_ptr(k), n, B, out.ctypes.data)
    return out


def doffset(mask) -> np.ndarray:
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    out = np.zeros(8 * m.size + 1, np.uint16)
    cnt = _load().orc_doffset(_ptr(m), m.size, out.ctypes.data)
    return out[:cnt].copy()


def popcount(mask) -> int:
    return int(np.unpackbits(np.asarray(mask, dtype=np.uint8)).sum())


def nplanes(m: int) -> int:
    return (m + 31) // 32


def compress(keys, mask, pext: bool = False) -> np.ndarray:
    """SoA planes uint32[ceil(m/32)][n] of P = Compress(key) (right-aligned)."""
    k = _keys(keys)
    n, B = k.shape
    mk = np.ascontiguousarray(mask, dtype=np.uint8)
    assert mk.size == B
    np_ = nplanes(popcount(mk))
    planes = np.zeros((np_, n), np.uint32)
    f = _load().orc_compress_pext if pext else _load().orc_compress
    f(_ptr(k), n, B, mk.ctypes.data, _ptr(planes))
    return planes


def pext_segments(mask):
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    st = np.zeros(m.size + 1, np.uint32)
    bits = np.zeros(m.size + 1, np.uint32)
    c = _load().orc_pext_segments(_ptr(m), m.size, st.ctypes.data, bits.ctypes.data)
    return st[:c].copy(), bits[:c].copy()


def sort_packed(planes, rid=None, threads: int = 1) -> np.ndarray:
    pl = np.ascontiguousarray(planes, dtype=np.uint32)
    np_, n = pl.shape
    perm = np.empty(n, np.uint32)
    r = None if rid is None else np.ascontiguousarray(rid, dtype=np.uint32)
    _load().orc_sort_packed(_ptr(pl), np_, n, _ptr(r), _ptr(perm), threads)
    return perm


def adjacent_compressed(sorted_planes, m: int, sort_mask):
    pl = np.ascontiguousarray(sorted_planes, dtype=np.uint32)
    n = pl.shape[1]
    sm = np.ascontiguousarray(sort_mask, dtype=np.uint8)
    dbit = np.empty(n, np.uint16)
    mask = np.zeros(sm.size, np.uint8)
    _load().orc_adjacent_compressed(_ptr(pl), m, n, sm.ctypes.data, sm.size, _ptr(dbit), mask.ctypes.data)
    return dbit, mask


def tree_levels(n: int, per: int) -> list[int]:
    lv, c = [], n
    if n == 0:
        return lv
    while True:
        c = (c + per - 1) // per
        lv.append(c)
        if c <= 1:
            return lv


def bulkload(perm, dbit, keys, fanout: int, fill: float = 1.0):
    """Dict with level_nodes, node_cnt, entry_rid, entry_child, entry_dbit."""
    k = _keys(keys)
    n, B = k.shape
    per = int(np.floor(fanout * fill))
    lv = tree_levels(n, per)
    total = int(sum(lv))
    perm = np.ascontiguousarray(perm, dtype=np.uint32)
    db = None if dbit is None else np.ascontiguousarray(dbit, dtype=np.uint16)
    level_nodes = np.zeros(max(1, len(lv)), np.uint64)
    node_cnt = np.zeros(total, np.uint32)
    rid = np.zeros((total, fanout), np.uint32)
    child = np.zeros((total, fanout), np.uint32)
    edb = np.zeros((total, fanout), np.uint16)
    h = _load().orc_bulkload(_ptr(perm), _ptr(db), n, fanout, per, _ptr(k), B,
                             level_nodes.ctypes.data, _ptr(node_cnt), _ptr(rid), _ptr(child), _ptr(edb))
    assert h == len(lv)
    return dict(height=h, level_nodes=level_nodes[:h].copy(), node_cnt=node_cnt,
                entry_rid=rid, entry_child=child, entry_dbit=edb, per=per)


def bulkload_blocks(perm, dbit, keys, block_n, fanout: int, fill: float = 1.0):
    """P:502 block-parallel construction (orc_bulkload_blocks): dict as bulkload()."""
    k = _keys(keys)
    n, B = k.shape
    per = int(np.floor(fanout * fill))
    bn = np.ascontiguousarray(np.asarray(block_n, dtype=np.uint64))
    assert int(bn.sum()) == n
    # node count bound: every block's levels + the top (at most n leaves + n inner overall)
    cap = max(1, 2 * n + 2 * len(bn) + 8)
    level_nodes = np.zeros(64, np.uint64)
    node_cnt = np.zeros(cap, np.uint32)
    rid = np.zeros((cap, fanout), np.uint32)
    child = np.zeros((cap, fanout), np.uint32)
    edb = np.zeros((cap, fanout), np.uint16)
    perm = np.ascontiguousarray(perm, dtype=np.uint32)
    db = None if dbit is None else np.ascontiguousarray(dbit, dtype=np.uint16)
    h = _load().orc_bulkload_blocks(_ptr(perm), _ptr(db), n, bn.ctypes.data, bn.size, fanout, per, _ptr(k), B,
                                    level_nodes.ctypes.data, _ptr(node_cnt), _ptr(rid), _ptr(child), _ptr(edb))
    total = int(level_nodes[:h].sum())
    return dict(height=h, level_nodes=level_nodes[:h].copy(), node_cnt=node_cnt[:total],
                entry_rid=rid[:total], entry_child=child[:total], entry_dbit=edb[:total], per=per)


def paper_tree_levels(n: int, leaf_per: int, inner_per: int) -> list[int]:
    """Nodes per level of the paper-format tree (leaves first)."""
    if n == 0:
        return []
    lv = [(n + leaf_per - 1) // leaf_per]
    while lv[-1] > 1:
        lv.append((lv[-1] + inner_per - 1) // inner_per)
    return lv


def paper_tree(keys, perm, dbit, pk: int = 32, fill: float = 0.9):
    """NEXT-3: node images u8[total][256] of the paper's index tree."""
    k = _keys(keys)
    n, B = k.shape
    leaf_per, inner_per = int(np.floor(14 * fill)), int(np.floor(9 * fill))
    lv = paper_tree_levels(n, leaf_per, inner_per)
    nodes = np.zeros((max(1, sum(lv)), 256), np.uint8)
    perm = np.ascontiguousarray(perm, dtype=np.uint32)
    db = np.ascontiguousarray(dbit, dtype=np.uint16)
    h = _load().orc_paper_tree(_ptr(k), n, B, _ptr(perm), _ptr(db), pk, leaf_per, inner_per, nodes.ctypes.data)
    assert h == len(lv)
    return dict(height=h, levels=lv, nodes=nodes[:sum(lv)], leaf_per=leaf_per, inner_per=inner_per)


def first_build(keys, threads: int = 1):
    """Full first build as the paper states it:
    exact D from the full-key sort, compress by D, sort (P, row id), D_i.
    Returns dict(mask, m, planes, perm, dbit)."""
    k = _keys(keys)
    perm = sort_keys(k, threads=threads)
    dbit, mask = adjacent_dbits(k, perm)
    planes = compress(k, mask)
    perm_p = sort_packed(planes, threads=threads)
    return dict(mask=mask, m=popcount(mask), planes=planes, perm=perm, perm_packed=perm_p, dbit=dbit)

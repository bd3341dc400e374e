"""Thin ctypes binding of libcks.so (include/cks.h). Argument marshalling only:
torch tensors provide device memory and the current CUDA stream; every step of the
path runs in the library's CUDA kernels. There is no CPU fallback -- if libcks.so is
missing or no CUDA device is present, calls raise.

Names follow the C ABI: superset_mask, distinction_mask, compress, sort,
adjacent_dbits, bulkload_shape, bulkload, build, build_host.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np
import torch

from . import _build

SO_PATH = _build.SO
CKS_OK, CKS_EINVAL, CKS_ERANGE, CKS_ENOMEM, CKS_ECUDA = 0, 1, 2, 3, 4
DBIT_NONE = 0xFFFF
MAX_LEVELS = 40
SUPERSET_VARIANT, SUPERSET_BYTEOCC = 0, 1

_lib = None
_lock = threading.Lock()
_ctx = {}


class CksError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"cks error {code}: {msg}")
        self.code = code


class TreeShape(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("fanout", ctypes.c_uint32), ("per_node", ctypes.c_uint32),
                ("height", ctypes.c_uint32), ("reserved", ctypes.c_uint32),
                ("level_nodes", ctypes.c_uint64 * MAX_LEVELS), ("level_offset", ctypes.c_uint64 * MAX_LEVELS),
                ("total_nodes", ctypes.c_uint64), ("inner_nodes", ctypes.c_uint64)]


class Tree(ctypes.Structure):
    _fields_ = [("node_cnt", ctypes.c_void_p), ("entry_rid", ctypes.c_void_p),
                ("entry_dbit", ctypes.c_void_p), ("entry_child", ctypes.c_void_p)]


class BuildOut(ctypes.Structure):
    _fields_ = [("mask", ctypes.c_void_p), ("perm", ctypes.c_void_p), ("dbit", ctypes.c_void_p),
                ("tree", Tree), ("fanout", ctypes.c_uint32), ("fill", ctypes.c_double),
                ("superset_kind", ctypes.c_int), ("popcount", ctypes.c_uint32),
                ("sort_bits", ctypes.c_uint32), ("height", ctypes.c_uint32), ("passes", ctypes.c_uint32),
                ("packed", ctypes.c_void_p), ("packed_pitch", ctypes.c_uint64),
                ("rounds", ctypes.c_uint32), ("round0_bits", ctypes.c_uint32), ("refined_keys", ctypes.c_uint64),
                ("variant", ctypes.c_void_p), ("ref_key", ctypes.c_void_p),
                ("ptree_nodes", ctypes.c_void_p), ("ptree_pk", ctypes.c_uint32), ("ptree_source", ctypes.c_uint32),
                ("ptree_fill", ctypes.c_double), ("sort_mask", ctypes.c_void_p)]


PTREE_AUTO, PTREE_ROWS, PTREE_DS, PTREE_CARRY, PTREE_DECODE = 0, 1, 2, 3, 4


EXPORTS = ["cks_ctx_create", "cks_ctx_destroy", "cks_ctx_set_stream", "cks_ctx_set_timing", "cks_ctx_set_sort_mode",
           "cks_ctx_stage_ms", "cks_ctx_launches", "cks_ctx_kernel_stats", "cks_strerror", "cks_last_error",
           "cks_superset_mask", "cks_distinction_mask", "cks_compress", "cks_sort",
           "cks_adjacent_dbits", "cks_bulkload_shape", "cks_bulkload", "cks_paper_tree_shape", "cks_paper_tree",
           "cks_build", "cks_build_host", "cks_occupancy", "cks_occupancy_mask", "cks_rank_sorted", "cks_repack",
           "cks_partition", "cks_sort_prefix", "cks_bulkload_block", "cks_bulkload_top",
           "cks_build_host_batch", "cks_ctx_set_round0_bits", "cks_ctx_set_verify",
           "cks_ctx_set_speculative_mask", "cks_ctx_speculation_stats", "cks_occupancy_sample",
           "cks_compress_marking",
           "cks_ctx_path_bytes", "cks_paper_tree_ds", "cks_partition_count", "cks_partition_send"]


def load_library(path: str | None = None):
    """Load libcks.so (raises if it was not built: run __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or SO_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"libcks.so not found at {path}; build it with `python __graft_entry__.py build`")
    L = ctypes.CDLL(path)
    p, u64, u32, i32, f32, f64 = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_float,
                                  ctypes.c_double)
    L.cks_ctx_create.argtypes = [i32, p, ctypes.POINTER(p)]
    L.cks_ctx_destroy.argtypes = [p]
    L.cks_ctx_set_stream.argtypes = [p, p]
    L.cks_ctx_set_timing.argtypes = [p, i32]
    L.cks_ctx_set_sort_mode.argtypes = [p, i32]
    L.cks_ctx_set_round0_bits.argtypes = [p, u32]
    L.cks_ctx_set_verify.argtypes = [p, i32]
    L.cks_ctx_set_speculative_mask.argtypes = [p, i32]
    L.cks_ctx_speculation_stats.argtypes = [p, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
    L.cks_ctx_path_bytes.argtypes = [p, ctypes.POINTER(ctypes.c_double)]
    L.cks_ctx_stage_ms.argtypes = [p, ctypes.POINTER(f32), i32]
    L.cks_ctx_launches.argtypes = [p]
    L.cks_ctx_launches.restype = u64
    L.cks_ctx_kernel_stats.argtypes = [p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(u32)]
    L.cks_strerror.argtypes = [i32]
    L.cks_strerror.restype = ctypes.c_char_p
    L.cks_last_error.argtypes = [p]
    L.cks_last_error.restype = ctypes.c_char_p
    L.cks_superset_mask.argtypes = [p, p, u64, u32, i32, p, ctypes.POINTER(u32)]
    L.cks_distinction_mask.argtypes = [p, p, u64, u32, p, p, ctypes.POINTER(u32), p]
    L.cks_compress.argtypes = [p, p, u64, u32, p, p]
    L.cks_sort.argtypes = [p, p, u32, u64, p, p, p]
    L.cks_adjacent_dbits.argtypes = [p, p, u32, u64, p, u32, p, ctypes.POINTER(u32), p]
    L.cks_bulkload_shape.argtypes = [u64, u32, f64, ctypes.POINTER(TreeShape)]
    L.cks_bulkload.argtypes = [p, p, p, u64, u32, f64, ctypes.POINTER(Tree)]
    L.cks_paper_tree_shape.argtypes = [u64, f64, ctypes.POINTER(TreeShape)]
    L.cks_paper_tree.argtypes = [p, p, u64, u32, p, p, u32, f64, p]
    L.cks_paper_tree_ds.argtypes = [p, p, u64, u32, p, p, p, u64, p, p, p, u32, f64, p]
    L.cks_build.argtypes = [p, p, u64, u32, p, ctypes.POINTER(BuildOut)]
    L.cks_build_host.argtypes = [p, p, u64, u32, p, ctypes.POINTER(BuildOut)]
    L.cks_occupancy.argtypes = [p, p, u64, u32, p]
    L.cks_occupancy_sample.argtypes = [p, p, u64, u32, u32, p]
    L.cks_compress_marking.argtypes = [p, p, u64, u32, p, p, p]
    L.cks_occupancy_mask.argtypes = [p, p, u32, u32, u64, i32, p, ctypes.POINTER(u32)]
    L.cks_rank_sorted.argtypes = [p, p, u32, u64, p, u64, p, u32, p]
    L.cks_repack.argtypes = [p, p, p, p, u32, u64, p]
    L.cks_partition.argtypes = [p, p, u32, u64, p, u32, u64, p, p, p]
    L.cks_partition_count.argtypes = [p, p, u32, u64, p, u32, u64, p]
    L.cks_partition_send.argtypes = [p, p, p, p]
    L.cks_sort_prefix.argtypes = [p, p, p, u32, u64, p, p, p, ctypes.POINTER(u32), p]
    L.cks_bulkload_block.argtypes = [p, p, p, u64, u32, f64, i32, u32, ctypes.POINTER(Tree), p, ctypes.POINTER(u32)]
    L.cks_bulkload_top.argtypes = [p, p, p, u64, u32, f64, ctypes.POINTER(Tree), ctypes.POINTER(u32)]
    L.cks_build_host_batch.argtypes = [p, p, u32, u64, u32, p, p]
    for name in EXPORTS:
        getattr(L, name).restype = getattr(L, name).restype or i32
    _lib = L
    return L


def _context(device: int | None = None):
    """The calling thread's context on `device` (one per (device, thread): a context owns
    scratch that its calls reuse, so threads driving one device each get their own)."""
    L = load_library()
    if not torch.cuda.is_available():
        raise RuntimeError("libcks needs a CUDA device (no CPU fallback)")
    dev = torch.cuda.current_device() if device is None else device
    key = (dev, threading.get_ident())
    with _lock:
        c = _ctx.get(key)
        if c is None:
            c = ctypes.c_void_p()
            stream = torch.cuda.current_stream(dev).cuda_stream
            rc = L.cks_ctx_create(dev, ctypes.c_void_p(stream), ctypes.byref(c))
            if rc != CKS_OK:
                raise CksError(rc, L.cks_strerror(rc).decode())
            _ctx[key] = c
    L.cks_ctx_set_stream(c, ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream))
    return L, c


def release_thread_contexts():
    """Destroy the calling thread's contexts (and their scratch)."""
    L = load_library()
    tid = threading.get_ident()
    with _lock:
        for key in [k for k in _ctx if k[1] == tid]:
            L.cks_ctx_destroy(_ctx.pop(key))


def _check(L, c, rc):
    if rc != CKS_OK:
        raise CksError(rc, f"{L.cks_strerror(rc).decode()}: {L.cks_last_error(c).decode()}")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _keys(keys: torch.Tensor):
    if keys.dtype != torch.uint8 or keys.dim() != 2 or not keys.is_cuda or not keys.is_contiguous():
        raise ValueError("keys must be a contiguous cuda uint8 tensor [n, key_bytes]")
    return keys.shape[0], keys.shape[1]


def _host_mask(mask, B: int) -> np.ndarray:
    m = np.ascontiguousarray(np.asarray(mask, dtype=np.uint8))
    if m.size != B:
        raise ValueError(f"mask must have {B} bytes")
    return m


def popcount(mask) -> int:
    return int(np.unpackbits(np.asarray(mask, dtype=np.uint8)).sum())


def nplanes(bits: int) -> int:
    return (bits + 31) // 32


def launches() -> int:
    L, c = _context()
    return int(L.cks_ctx_launches(c))


def set_timing(enable: bool):
    L, c = _context()
    L.cks_ctx_set_timing(c, 1 if enable else 0)


SORT_SINGLE, SORT_PREFIX_AUTO, SORT_PREFIX = 0, 1, 2


def set_sort_mode(mode: int, device: int | None = None):
    """CKS_SORT_SINGLE / CKS_SORT_PREFIX_AUTO (default) / CKS_SORT_PREFIX for later builds."""
    L, c = _context(device)
    _check(L, c, L.cks_ctx_set_sort_mode(c, int(mode)))


def set_round0_bits(bits: int, device: int | None = None):
    """Width of refinement round 0 for later builds (0 = sampled; else a multiple of 8 <= 64)."""
    L, c = _context(device)
    _check(L, c, L.cks_ctx_set_round0_bits(c, int(bits)))


VERIFY_OFF, VERIFY_PRIOR, VERIFY_ALWAYS = 0, 1, 2


def set_verify(mode: int, device: int | None = None):
    """Order check of later builds against the key rows (cks_ctx_set_verify)."""
    L, c = _context(device)
    _check(L, c, L.cks_ctx_set_verify(c, int(mode)))


def set_speculative_mask(enable: bool, device: int | None = None):
    """First builds take the mask from a row sample and let the compress mark the occupancy
    (default on; cks_ctx_set_speculative_mask)."""
    L, c = _context(device)
    _check(L, c, L.cks_ctx_set_speculative_mask(c, 1 if enable else 0))


def speculation_stats(device: int | None = None) -> tuple[int, int]:
    """(speculative first builds, of them rebuilt by the full D+) on this thread's context."""
    L, c = _context(device)
    b, r = ctypes.c_uint64(), ctypes.c_uint64()
    _check(L, c, L.cks_ctx_speculation_stats(c, ctypes.byref(b), ctypes.byref(r)))
    return int(b.value), int(r.value)


def stage_ms() -> list[float]:
    L, c = _context()
    buf = (ctypes.c_float * 8)()
    k = L.cks_ctx_stage_ms(c, buf, 8)
    return [float(buf[i]) for i in range(k)]


def kernel_stats() -> tuple[float, float, int]:
    """(ms, algorithmic bytes, launches) of the dominant kernel in the last timed build."""
    L, c = _context()
    ms, by, cnt = ctypes.c_double(), ctypes.c_double(), ctypes.c_uint32()
    _check(L, c, L.cks_ctx_kernel_stats(c, ctypes.byref(ms), ctypes.byref(by), ctypes.byref(cnt)))
    return float(ms.value), float(by.value), int(cnt.value)


def path_bytes() -> float:
    """Algorithmic bytes of every kernel of the last build on this thread's context."""
    L, c = _context()
    b = ctypes.c_double()
    _check(L, c, L.cks_ctx_path_bytes(c, ctypes.byref(b)))
    return float(b.value)


def superset_mask(keys: torch.Tensor, kind: int = SUPERSET_BYTEOCC) -> np.ndarray:
    n, B = _keys(keys)
    L, c = _context(keys.device.index)
    mask = np.zeros(B, np.uint8)
    pc = ctypes.c_uint32()
    _check(L, c, L.cks_superset_mask(c, _ptr(keys), n, B, kind, mask.ctypes.data, ctypes.byref(pc)))
    return mask


def distinction_mask(keys: torch.Tensor, prior_mask=None, want_perm: bool = True):
    """(exact D mask [B] uint8, perm tensor or None)."""
    n, B = _keys(keys)
    L, c = _context(keys.device.index)
    mask = np.zeros(B, np.uint8)
    pm = None if prior_mask is None else _host_mask(prior_mask, B)
    perm = torch.empty(n, dtype=torch.int32, device=keys.device) if want_perm else None
    pc = ctypes.c_uint32()
    _check(L, c, L.cks_distinction_mask(c, _ptr(keys), n, B, None if pm is None else pm.ctypes.data,
                                        mask.ctypes.data, ctypes.byref(pc), _ptr(perm)))
    return mask, perm


def compress(keys: torch.Tensor, mask) -> torch.Tensor:
    """SoA planes int32[ceil(m/32)][n] (bit patterns of u32) of Compress_mask(key)."""
    n, B = _keys(keys)
    L, c = _context(keys.device.index)
    m = _host_mask(mask, B)
    out = torch.empty((nplanes(popcount(m)), n), dtype=torch.int32, device=keys.device)
    _check(L, c, L.cks_compress(c, _ptr(keys), n, B, m.ctypes.data, _ptr(out) if out.numel() else None))
    return out


def sort(packed: torch.Tensor, bits: int, row_ids: torch.Tensor | None = None, want_sorted: bool = False):
    """(perm int32[n], sorted planes or None)."""
    n = packed.shape[1]
    L, c = _context(packed.device.index)
    if packed.dtype != torch.int32 or not packed.is_contiguous() or packed.shape[0] != nplanes(bits):
        raise ValueError("packed must be contiguous int32 [ceil(bits/32), n]")
    perm = torch.empty(n, dtype=torch.int32, device=packed.device)
    srt = torch.empty_like(packed) if want_sorted else None
    if row_ids is not None and (row_ids.dtype != torch.int32 or row_ids.numel() != n):
        raise ValueError("row_ids must be int32 [n]")
    _check(L, c, L.cks_sort(c, _ptr(packed) if packed.numel() else None, bits, n, _ptr(row_ids), _ptr(perm),
                            _ptr(srt) if srt is not None and srt.numel() else None))
    return perm, srt


def adjacent_dbits(sorted_packed: torch.Tensor, bits: int, sort_mask, want_dbit: bool = True):
    """(exact D mask [B], dbit int16[n] or None) from sorted planes."""
    n = sorted_packed.shape[1]
    sm = np.ascontiguousarray(np.asarray(sort_mask, dtype=np.uint8))
    B = sm.size
    L, c = _context(sorted_packed.device.index)
    mask = np.zeros(B, np.uint8)
    dbit = torch.empty(n, dtype=torch.int16, device=sorted_packed.device) if want_dbit else None
    pc = ctypes.c_uint32()
    _check(L, c, L.cks_adjacent_dbits(c, _ptr(sorted_packed) if sorted_packed.numel() else None, bits, n,
                                      sm.ctypes.data, B, mask.ctypes.data, ctypes.byref(pc), _ptr(dbit)))
    return mask, dbit


# ---- NEXT-4: per-shard steps of the sharded path (shard.py drives them) -------------------

def occupancy(keys: torch.Tensor) -> torch.Tensor:
    """int32[B*8] (u32 bit patterns): per-byte occupancy of these keys (cks_occupancy)."""
    n, B = _keys(keys)
    L, c = _context(keys.device.index)
    occ = torch.empty(B * 8, dtype=torch.int32, device=keys.device)
    _check(L, c, L.cks_occupancy(c, _ptr(keys), n, B, _ptr(occ)))
    return occ


def occupancy_sample(keys: torch.Tensor, samples: int) -> torch.Tensor:
    """int32[B*8]: occupancy of `samples` rows strided over these keys (cks_occupancy_sample)."""
    n, B = _keys(keys)
    L, c = _context(keys.device.index)
    occ = torch.empty(B * 8, dtype=torch.int32, device=keys.device)
    _check(L, c, L.cks_occupancy_sample(c, _ptr(keys), n, B, int(samples), _ptr(occ)))
    return occ


def compress_marking(keys: torch.Tensor, mask):
    """(P planes as compress(), int32[B*8] occupancy of all these keys) from one read of the
    keys (cks_compress_marking)."""
    n, B = _keys(keys)
    L, c = _context(keys.device.index)
    m = _host_mask(mask, B)
    out = torch.empty((nplanes(popcount(m)), n), dtype=torch.int32, device=keys.device)
    occ = torch.empty(B * 8, dtype=torch.int32, device=keys.device)
    _check(L, c, L.cks_compress_marking(c, _ptr(keys), n, B, m.ctypes.data, _ptr(out) if out.numel() else None,
                                        _ptr(occ)))
    return out, occ


def marks_occupancy(keys: torch.Tensor) -> bool:
    """Whether compress_marking applies (16-byte aligned keys of 8/16/32/64 bytes)."""
    return keys.shape[1] in (8, 16, 32, 64) and keys.data_ptr() % 16 == 0


def occupancy_mask(occs: torch.Tensor, n_total: int, kind: int = SUPERSET_BYTEOCC) -> np.ndarray:
    """Superset mask [B] of the union of stacked occupancies int32[G, B*8] (cks_occupancy_mask)."""
    if occs.dtype != torch.int32 or occs.dim() != 2 or occs.shape[1] % 8 or not occs.is_contiguous():
        raise ValueError("occs must be contiguous int32 [G, B*8]")
    G, B = occs.shape[0], occs.shape[1] // 8
    L, c = _context(occs.device.index)
    mask = np.zeros(B, np.uint8)
    pc = ctypes.c_uint32()
    _check(L, c, L.cks_occupancy_mask(c, _ptr(occs), G, B, n_total, kind, mask.ctypes.data, ctypes.byref(pc)))
    return mask


def rank_sorted(sorted_packed: torch.Tensor, bits: int, sorted_rid: torch.Tensor, rid_base: int,
                queries: torch.Tensor) -> torch.Tensor:
    """int64[nq]: lower-bound ranks of (P, row id) queries int32[nq, np+1] in a sorted shard."""
    n = sorted_packed.shape[1]
    nq = queries.shape[0]
    if queries.dtype != torch.int32 or not queries.is_contiguous() or queries.shape[1] != nplanes(bits) + 1:
        raise ValueError("queries must be contiguous int32 [nq, ceil(bits/32)+1]")
    L, c = _context(sorted_packed.device.index)
    ranks = torch.empty(nq, dtype=torch.int64, device=sorted_packed.device)
    _check(L, c, L.cks_rank_sorted(c, _ptr(sorted_packed) if sorted_packed.numel() else None, bits, n,
                                   _ptr(sorted_rid), rid_base, _ptr(queries) if nq else None, nq,
                                   _ptr(ranks) if nq else None))
    return ranks


def partition(packed: torch.Tensor, bits: int, splitters: torch.Tensor, parts: int, rid_base: int):
    """(packed int32[np, n], row ids int32[n], counts int64[parts]): stable partition of the
    (P, rid_base + i) pairs by parts-1 splitters int32[parts-1, np+1] (cks_partition)."""
    n = packed.shape[1]
    if packed.dtype != torch.int32 or not packed.is_contiguous() or packed.shape[0] != nplanes(bits):
        raise ValueError("packed must be contiguous int32 [ceil(bits/32), n]")
    if splitters.dtype != torch.int32 or not splitters.is_contiguous() or splitters.shape[0] != parts - 1:
        raise ValueError("splitters must be contiguous int32 [parts-1, ceil(bits/32)+1]")
    L, c = _context(packed.device.index)
    out = torch.empty_like(packed)
    rid = torch.empty(n, dtype=torch.int32, device=packed.device)
    counts = torch.empty(parts, dtype=torch.int64, device=packed.device)
    _check(L, c, L.cks_partition(c, _ptr(packed) if packed.numel() else None, bits, n,
                                 _ptr(splitters) if splitters.numel() else None, parts, rid_base,
                                 _ptr(out) if out.numel() else None, _ptr(rid) if n else None, _ptr(counts)))
    return out, rid, counts


def partition_count(packed: torch.Tensor, bits: int, splitters: torch.Tensor, parts: int, rid_base: int):
    """int64[parts]: elements per part of the stable partition by parts-1 splitters (the first
    half of the fused partition-and-send, cks_partition_count)."""
    n = packed.shape[1]
    if packed.dtype != torch.int32 or not packed.is_contiguous() or packed.shape[0] != nplanes(bits):
        raise ValueError("packed must be contiguous int32 [ceil(bits/32), n]")
    if splitters.dtype != torch.int32 or not splitters.is_contiguous() or splitters.shape[0] != parts - 1:
        raise ValueError("splitters must be contiguous int32 [parts-1, ceil(bits/32)+1]")
    L, c = _context(packed.device.index)
    counts = torch.empty(parts, dtype=torch.int64, device=packed.device)
    _check(L, c, L.cks_partition_count(c, _ptr(packed) if packed.numel() else None, bits, n,
                                       _ptr(splitters) if splitters.numel() else None, parts, rid_base,
                                       _ptr(counts)))
    return counts


def partition_send(dst_planes: list, dst_pitch: list, dst_rid: list, device: int | None = None):
    """Second half (cks_partition_send): write every part of the last partition_count on this
    thread's context straight into its receiver's buffers (device addresses, element units:
    dst_planes[d] + q * dst_pitch[d] is plane q of part d's destination)."""
    L, c = _context(device)
    k = len(dst_rid)
    P = ctypes.c_void_p * k
    pit = (ctypes.c_uint64 * k)(*[int(x) for x in dst_pitch])
    _check(L, c, L.cks_partition_send(c, P(*dst_planes), pit, P(*dst_rid)))


def sort_prefix(packed: torch.Tensor, sort_mask, want_packed: bool = False):
    """(order int32[n], dbit int16[n], exact D [B], P_D int32[.., n] or None): the first build's
    sort by distinguishing prefixes on given P_M planes int32[ceil(m/32), n] (cks_sort_prefix)."""
    sm = np.ascontiguousarray(np.asarray(sort_mask, dtype=np.uint8))
    B = sm.size
    n = packed.shape[1]
    if packed.dtype != torch.int32 or not packed.is_contiguous() or packed.shape[0] != nplanes(popcount(sm)):
        raise ValueError("packed must be contiguous int32 [ceil(m/32), n]")
    L, c = _context(packed.device.index)
    order = torch.empty(n, dtype=torch.int32, device=packed.device)
    dbit = torch.empty(n, dtype=torch.int16, device=packed.device)
    mask = np.zeros(B, np.uint8)
    pc = ctypes.c_uint32()
    out = None
    if want_packed:
        out = torch.empty((0, n), dtype=torch.int32, device=packed.device)
    # P_D's width is known only after the sort: size it for |M| planes, trim after
    buf = torch.empty((packed.shape[0], n), dtype=torch.int32, device=packed.device) if want_packed else None
    _check(L, c, L.cks_sort_prefix(c, _ptr(packed) if packed.numel() else None, sm.ctypes.data, B, n,
                                   _ptr(order) if n else None, _ptr(dbit) if n else None, mask.ctypes.data,
                                   ctypes.byref(pc), _ptr(buf) if buf is not None and buf.numel() else None))
    if want_packed:
        out = buf[:nplanes(int(pc.value))]
    return order, dbit, mask, out


def repack(packed: torch.Tensor, in_mask, out_mask) -> torch.Tensor:
    """P_out (int32[ceil(|out|/32), n]) from P_in for out_mask a subset of in_mask (cks_repack)."""
    im = np.ascontiguousarray(np.asarray(in_mask, dtype=np.uint8))
    om = np.ascontiguousarray(np.asarray(out_mask, dtype=np.uint8))
    n = packed.shape[1]
    L, c = _context(packed.device.index)
    out = torch.empty((nplanes(popcount(om)), n), dtype=torch.int32, device=packed.device)
    _check(L, c, L.cks_repack(c, _ptr(packed) if packed.numel() else None, im.ctypes.data, om.ctypes.data, im.size, n,
                              _ptr(out) if out.numel() else None))
    return out


def bulkload_shape(n: int, fanout: int, fill: float = 1.0) -> TreeShape:
    s = TreeShape()
    rc = load_library().cks_bulkload_shape(n, fanout, fill, ctypes.byref(s))
    if rc != CKS_OK:
        raise CksError(rc, "bad bulk-load shape")
    return s


def alloc_tree(shape: TreeShape, device, with_dbit: bool = True, with_child: bool = True) -> dict:
    T, f = int(shape.total_nodes), int(shape.fanout)
    return dict(
        node_cnt=torch.empty(max(T, 1), dtype=torch.int32, device=device),
        entry_rid=torch.empty(max(T * f, 1), dtype=torch.int32, device=device),
        entry_dbit=torch.empty(max(T * f, 1), dtype=torch.int16, device=device) if with_dbit else None,
        entry_child=torch.empty(max(int(shape.inner_nodes) * f, 1), dtype=torch.int32, device=device)
        if with_child else None)


def _tree_struct(t: dict) -> Tree:
    return Tree(t["node_cnt"].data_ptr(), t["entry_rid"].data_ptr(),
                t["entry_dbit"].data_ptr() if t.get("entry_dbit") is not None else None,
                t["entry_child"].data_ptr() if t.get("entry_child") is not None else None)


def bulkload(perm: torch.Tensor, dbit: torch.Tensor | None, fanout: int = 64, fill: float = 1.0,
             with_child: bool = True) -> dict:
    n = perm.numel()
    L, c = _context(perm.device.index)
    shape = bulkload_shape(n, fanout, fill)
    t = alloc_tree(shape, perm.device, with_dbit=dbit is not None, with_child=with_child)
    tr = _tree_struct(t)
    _check(L, c, L.cks_bulkload(c, _ptr(perm), _ptr(dbit), n, fanout, fill, ctypes.byref(tr)))
    t["shape"] = shape
    return t


def bulkload_block(perm: torch.Tensor, dbit: torch.Tensor, fanout: int, fill: float, first_global: bool,
                   levels: int = 0) -> dict:
    """P:502 subtree over one block (cks_bulkload_block): tree dict of the block's levels
    0..levels-1 plus "top_min" (minimum D_k under each node of the top built level) and
    "height" (levels built)."""
    n = perm.numel()
    L, c = _context(perm.device.index)
    shape = bulkload_shape(n, fanout, fill)
    t = alloc_tree(shape, perm.device, with_dbit=True, with_child=True)
    tr = _tree_struct(t)
    H = min(levels, int(shape.height)) if levels else int(shape.height)
    top_min = torch.empty(max(1, int(shape.level_nodes[H - 1]) if H else 1), dtype=torch.int16, device=perm.device)
    h = ctypes.c_uint32()
    _check(L, c, L.cks_bulkload_block(c, _ptr(perm) if n else None, _ptr(dbit) if n else None, n, fanout, fill,
                                      1 if first_global else 0, levels, ctypes.byref(tr),
                                      _ptr(top_min) if n else None, ctypes.byref(h)))
    t["shape"], t["height"], t["top_min"] = shape, int(h.value), top_min
    return t


def bulkload_top(child_rid: torch.Tensor, child_min: torch.Tensor, fanout: int, fill: float) -> dict:
    """P:502 merged top over the blocks' top nodes (cks_bulkload_top)."""
    nc = child_rid.numel()
    L, c = _context(child_rid.device.index)
    shape = bulkload_shape(nc, fanout, fill)
    T = int(shape.total_nodes) if nc > 1 else 0
    f = fanout
    t = dict(node_cnt=torch.empty(max(T, 1), dtype=torch.int32, device=child_rid.device),
             entry_rid=torch.empty(max(T * f, 1), dtype=torch.int32, device=child_rid.device),
             entry_dbit=torch.empty(max(T * f, 1), dtype=torch.int16, device=child_rid.device),
             entry_child=torch.empty(max(T * f, 1), dtype=torch.int32, device=child_rid.device))
    tr = _tree_struct(t)
    h = ctypes.c_uint32()
    _check(L, c, L.cks_bulkload_top(c, _ptr(child_rid) if nc else None, _ptr(child_min) if nc else None, nc, fanout,
                                    fill, ctypes.byref(tr), ctypes.byref(h)))
    t["height"], t["nodes"] = int(h.value), T
    return t


PTREE_NODE_BYTES = 256


def paper_tree_shape(n: int, fill: float = 0.9) -> TreeShape:
    """NEXT-3 tree shape: per_node = leaf entries, reserved = non-leaf entries."""
    s = TreeShape()
    rc = load_library().cks_paper_tree_shape(n, fill, ctypes.byref(s))
    if rc != CKS_OK:
        raise CksError(rc, "bad paper-tree shape")
    return s


def paper_tree(keys: torch.Tensor, perm: torch.Tensor, dbit: torch.Tensor, pk_bits: int = 32,
               fill: float = 0.9, out: torch.Tensor | None = None) -> torch.Tensor:
    """NEXT-3: the paper's 256-byte-node index tree (include/cks.h layout) as u8[total][256]."""
    n, B = _keys(keys)
    L, c = _context(keys.device.index)
    s = paper_tree_shape(n, fill)
    T = int(s.total_nodes)
    if out is None:
        out = torch.empty((max(T, 1), PTREE_NODE_BYTES), dtype=torch.uint8, device=keys.device)
    _check(L, c, L.cks_paper_tree(c, _ptr(keys), n, B, _ptr(perm), _ptr(dbit), pk_bits, fill, _ptr(out)))
    return out[:T]


def paper_tree_ds(keys: torch.Tensor | None, n: int, B: int, perm: torch.Tensor, dbit: torch.Tensor,
                  packed: torch.Tensor | None, packed_pitch: int, packed_mask, variant, ref_key, pk_bits: int = 32,
                  fill: float = 0.9, out: torch.Tensor | None = None) -> torch.Tensor:
    """NEXT-3 tree with partial keys from the DS-metadata sources (cks_paper_tree_ds): packed =
    the sorted compressed planes (int32 [.., >= n], row pitch packed_pitch) of packed_mask."""
    dev = perm.device
    L, c = _context(dev.index)
    s = paper_tree_shape(n, fill)
    T = int(s.total_nodes)
    if out is None:
        out = torch.empty((max(T, 1), PTREE_NODE_BYTES), dtype=torch.uint8, device=dev)
    xm, vm, rk = _host_mask(packed_mask, B), _host_mask(variant, B), _host_mask(ref_key, B)
    _check(L, c, L.cks_paper_tree_ds(c, _ptr(keys), n, B, _ptr(perm), _ptr(dbit),
                                     _ptr(packed) if packed is not None and packed.numel() else None, packed_pitch,
                                     xm.ctypes.data, vm.ctypes.data, rk.ctypes.data, pk_bits, fill, _ptr(out)))
    return out[:T]


class Builder:
    """Preallocated fused first build (cks_build) for repeated steps on one key shape."""

    def __init__(self, n: int, B: int, device, fanout: int = 64, fill: float = 1.0,
                 superset_kind: int = SUPERSET_BYTEOCC, tree: bool = True, dbit: bool = True,
                 ds_metadata: bool = False, paper_tree_pk: int | None = None, paper_tree_fill: float = 0.9,
                 paper_tree_source: int = 0):
        self.n, self.B = n, B
        self.mask = np.zeros(B, np.uint8)
        self.sort_mask = np.zeros(B, np.uint8)                   # the mask the sort ran on
        # DS-metadata: variant bitmap and reference key, recomputed by the build
        self.variant = np.zeros(B, np.uint8) if ds_metadata else None
        self.ref_key = np.zeros(B, np.uint8) if ds_metadata else None
        self.perm = torch.empty(max(n, 1), dtype=torch.int32, device=device)
        self.dbit = torch.empty(max(n, 1), dtype=torch.int16, device=device) if dbit else None
        self.shape = bulkload_shape(n, fanout, fill)
        self.tree = alloc_tree(self.shape, device) if tree else None
        self.out = BuildOut()
        self.out.mask = self.mask.ctypes.data
        self.out.sort_mask = self.sort_mask.ctypes.data
        self.out.perm = self.perm.data_ptr()
        self.out.dbit = self.dbit.data_ptr() if self.dbit is not None else None
        if self.tree is not None:
            self.out.tree = _tree_struct(self.tree)
        self.out.fanout = fanout
        self.out.fill = fill
        self.out.superset_kind = superset_kind
        if ds_metadata:
            self.out.variant = self.variant.ctypes.data
            self.out.ref_key = self.ref_key.ctypes.data
        # NEXT-3: the paper-format tree built by the same call (partial keys from A/B/C(a))
        self.ptree = None
        if paper_tree_pk is not None:
            ps = paper_tree_shape(n, paper_tree_fill)
            self.ptree = torch.empty((max(int(ps.total_nodes), 1), PTREE_NODE_BYTES), dtype=torch.uint8,
                                     device=device)
            self.ptree_nodes = int(ps.total_nodes)
            self.out.ptree_nodes = self.ptree.data_ptr()
            self.out.ptree_pk = paper_tree_pk
            self.out.ptree_fill = paper_tree_fill
            self.out.ptree_source = paper_tree_source

    def __call__(self, keys: torch.Tensor, prior_mask=None) -> "Builder":
        n, B = _keys(keys)
        assert (n, B) == (self.n, self.B)
        L, c = _context(keys.device.index)
        pm = None if prior_mask is None else _host_mask(prior_mask, B)
        _check(L, c, L.cks_build(c, _ptr(keys), n, B, None if pm is None else pm.ctypes.data,
                                 ctypes.byref(self.out)))
        return self

    def packed(self) -> torch.Tensor | None:
        """Copy of the sorted P_D planes (ctx-owned view -> new tensor)."""
        npd = nplanes(int(self.out.popcount))
        if npd == 0 or self.n == 0:
            return torch.empty((0, self.n), dtype=torch.int32, device=self.perm.device)
        pitch = int(self.out.packed_pitch)
        src = raw_view(int(self.out.packed), npd * pitch, self.perm.device).view(npd, pitch)
        return src[:, :self.n].clone()


def raw_view(ptr: int, numel: int, device) -> torch.Tensor:
    """int32 tensor view of library-owned device memory (valid until the next call)."""
    class _View:
        __cuda_array_interface__ = {"shape": (numel,), "typestr": "<i4", "data": (ptr, False),
                                    "version": 3, "strides": None, "stream": None}
    return torch.as_tensor(_View(), device=device)


def build(keys: torch.Tensor, prior_mask=None, fanout: int = 64, fill: float = 1.0,
          superset_kind: int = SUPERSET_BYTEOCC, tree: bool = True, ds_metadata: bool = False,
          paper_tree_pk: int | None = None, paper_tree_fill: float = 0.9, paper_tree_source: int = 0) -> dict:
    n, B = _keys(keys)
    b = Builder(n, B, keys.device, fanout, fill, superset_kind, tree, ds_metadata=ds_metadata,
                paper_tree_pk=paper_tree_pk, paper_tree_fill=paper_tree_fill, paper_tree_source=paper_tree_source)
    b(keys, prior_mask)
    o = b.out
    r = dict(mask=b.mask.copy(), popcount=int(o.popcount), sort_bits=int(o.sort_bits), sort_mask=b.sort_mask.copy(),
             passes=int(o.passes),
             perm=b.perm[:n], dbit=b.dbit[:n] if b.dbit is not None else None, packed=b.packed(),
             tree=b.tree, shape=b.shape, height=int(o.height))
    if ds_metadata:
        r.update(variant=b.variant.copy(), ref_key=b.ref_key.copy())
    if b.ptree is not None:
        r["paper_tree"] = b.ptree[:b.ptree_nodes]
    return r


def build_host_batch(columns: list, prior_mask=None, superset_kind: int = SUPERSET_BYTEOCC,
                     perms: list | None = None, device: int | None = None) -> list[dict]:
    """Pipelined fused builds of several HOST key columns (numpy uint8 [n, B] each, same shape,
    ideally pinned): copies, builds and result copies overlap (cks_build_host_batch)."""
    cols = [np.ascontiguousarray(c) for c in columns]
    if not cols:
        return []
    n, B = cols[0].shape
    if any(c.dtype != np.uint8 or c.shape != (n, B) for c in cols):
        raise ValueError("columns must be uint8 [n, B] of one shape")
    L, c = _context(device)
    k = len(cols)
    masks = [np.zeros(B, np.uint8) for _ in range(k)]
    perms = perms if perms is not None else [np.empty(n, np.uint32) for _ in range(k)]
    outs = (BuildOut * k)()
    for i in range(k):
        outs[i].mask = masks[i].ctypes.data
        outs[i].perm = perms[i].ctypes.data
        outs[i].superset_kind = superset_kind
        outs[i].fanout, outs[i].fill = 64, 1.0
    ptrs = (ctypes.c_void_p * k)(*[x.ctypes.data if n else None for x in cols])
    pm = None if prior_mask is None else _host_mask(prior_mask, B)
    _check(L, c, L.cks_build_host_batch(c, ptrs, k, n, B, None if pm is None else pm.ctypes.data, outs))
    return [dict(mask=masks[i], popcount=int(outs[i].popcount), sort_bits=int(outs[i].sort_bits), perm=perms[i])
            for i in range(k)]


def build_host(host_keys: np.ndarray, prior_mask=None, superset_kind: int = SUPERSET_BYTEOCC,
               perm_out: np.ndarray | None = None, device: int | None = None) -> dict:
    """Fused build from HOST keys (numpy uint8 [n, B], ideally pinned) -> host perm."""
    k = np.ascontiguousarray(host_keys)
    if k.dtype != np.uint8 or k.ndim != 2:
        raise ValueError("host_keys must be uint8 [n, B]")
    n, B = k.shape
    L, c = _context(device)
    mask = np.zeros(B, np.uint8)
    perm = perm_out if perm_out is not None else np.empty(n, np.uint32)
    o = BuildOut()
    o.mask = mask.ctypes.data
    o.perm = perm.ctypes.data
    o.superset_kind = superset_kind
    o.fanout, o.fill = 64, 1.0
    pm = None if prior_mask is None else _host_mask(prior_mask, B)
    _check(L, c, L.cks_build_host(c, k.ctypes.data if n else None, n, B, None if pm is None else pm.ctypes.data,
                                  ctypes.byref(o)))
    return dict(mask=mask, popcount=int(o.popcount), sort_bits=int(o.sort_bits), perm=perm)

"""NEXT-4: the sharded first build.

One rank per GPU holds a contiguous shard of the key column (rank r: global row ids
off_r .. off_r + n_r - 1). The method shards with one exchange step:

  a1  per-shard byte occupancy -> all-gather -> union -> D+ (cks_occupancy[_mask]); NCCL has
      no bitwise-OR reduction, so the union is taken on the gathered occupancies;
  a3  compress the shard by D+ (row-parallel, no exchange);
  a5  a regular sample of every shard -> all-gather -> G-1 splitters in the (P, row id)
      order (total: duplicates split by row id); every shard is partitioned by them, stably
      (cks_partition: one destination pass + one digit pass) -> ONE all-to-all of
      (P, row id); the received parts, concatenated in source-rank order, are in row-id
      order, so one stable sort on P alone orders them by (P, row id): rank r now holds the
      r-th slice of the global order (the paper's range partition);
  a6  adjacency over the slice plus the pair across each slice boundary (the previous
      non-empty slice's last key is all-gathered), D = OR of the slices' D (all-gather);
  a7  P_D of the slice by repacking P_{D+} (cks_repack);
  a8  P:502: every rank bulk-loads a subtree over its slice (cks_bulkload_block), the
      subtrees' roots are removed and rank 0 builds the top layers over the roots' children
      (cks_bulkload_top); the tree stays distributed (assemble_tree joins it on the host).

Every per-shard step is a libcks kernel (`CudaOps`); this module only moves data between
ranks. `Comm` implementations: `TorchComm` (torch.distributed: NCCL between GPUs, gloo for
the CPU tests) and `ThreadComm` (G ranks as threads of one process on one device -- no
kernel waits on another rank; used to run the sharded path on one GPU).
"""
from __future__ import annotations

import threading

import numpy as np
import torch

from . import cks

NONE = 0xFFFF


# ---- communicators -----------------------------------------------------------------------

class TorchComm:
    """Collectives over a torch.distributed process group (NCCL: CUDA tensors; gloo: the
    tensors are staged through host memory). Peer buffers for the fused partition-and-send are
    shared as CUDA IPC handles (torch.multiprocessing's reduction of a CUDA tensor: the peer
    maps the owner's allocation; across GPUs the kernel's stores go over NVLink); peer_access =
    False falls back to the partition + all-to-all baseline."""
    peer_access = True

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.cpu = dist.get_backend(group) == "gloo"

    def _dev(self, t):
        return t.cpu() if self.cpu else t

    def allgather(self, t: torch.Tensor) -> list[torch.Tensor]:
        x = self._dev(t.contiguous())
        out = [torch.empty_like(x) for _ in range(self.size)]
        self.dist.all_gather(out, x, group=self.group)
        return [o.to(t.device) for o in out]

    def peer_tensors(self, tensors: tuple) -> list[tuple]:
        """Every rank's `tensors` (CUDA), usable from this process: own rank as is, the others
        opened from their CUDA IPC handles."""
        from torch.multiprocessing.reductions import reduce_tensor
        torch.cuda.current_stream().synchronize()
        mine = [reduce_tensor(t) for t in tensors]
        objs = [None] * self.size
        self.dist.all_gather_object(objs, mine, group=self.group)
        out = []
        for d, o in enumerate(objs):
            out.append(tuple(tensors) if d == self.rank else tuple(fn(*args) for fn, args in o))
        return out

    def barrier(self):
        torch.cuda.current_stream().synchronize()
        self.dist.barrier(group=self.group)

    def alltoallv(self, t: torch.Tensor, send_counts: list[int], recv_counts: list[int] | None = None) -> torch.Tensor:
        """Rows [sum(send_counts[:d]), +send_counts[d]) of t go to rank d; returns the rows
        received, source rank order. recv_counts (known from the all-gathered count matrix)
        saves the count exchange."""
        x = self._dev(t.contiguous())
        if recv_counts is None:
            sc = torch.tensor(send_counts, dtype=torch.int64)
            rc = torch.empty_like(sc)
            sc_d, rc_d = (sc, rc) if self.cpu else (sc.to(t.device), rc.to(t.device))
            self.dist.all_to_all_single(rc_d, sc_d, group=self.group)
            recv_counts = [int(v) for v in rc_d.tolist()]
        out = torch.empty((sum(recv_counts),) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        self.dist.all_to_all_single(out, x, recv_counts, send_counts, group=self.group)
        return out.to(t.device)


class ThreadComm:
    """G ranks as threads of one process (each thread: its own CUDA stream and libcks
    context). A collective synchronises the caller's stream, publishes its tensor, and
    waits at a barrier for the others."""

    class _Shared:
        def __init__(self, size):
            self.size = size
            self.barrier = threading.Barrier(size)
            self.slots = [None] * size

    peer_access = True                   # all ranks on one device: a rank may write another's buffers

    def __init__(self, shared, rank):
        self.sh, self.rank, self.size = shared, rank, shared.size

    @classmethod
    def group(cls, size: int) -> list["ThreadComm"]:
        sh = cls._Shared(size)
        return [cls(sh, r) for r in range(size)]

    def _publish(self, obj):
        if torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()
        self.sh.slots[self.rank] = obj
        self.sh.barrier.wait()

    def allgather(self, t: torch.Tensor) -> list[torch.Tensor]:
        self._publish(t.contiguous())
        out = [s.clone() for s in self.sh.slots]
        self.sh.barrier.wait()
        return out

    def allgather_obj(self, obj) -> list:
        self._publish(obj)
        out = list(self.sh.slots)
        self.sh.barrier.wait()
        return out

    def barrier(self):
        self.allgather_obj(None)

    def peer_tensors(self, tensors: tuple) -> list[tuple]:
        """Every rank's `tensors` (all ranks share the device and the address space)."""
        return self.allgather_obj(tuple(tensors))

    def alltoallv(self, t: torch.Tensor, send_counts: list[int], recv_counts: list[int] | None = None) -> torch.Tensor:
        self._publish(list(torch.split(t.contiguous(), send_counts, dim=0)))
        out = torch.cat([self.sh.slots[s][self.rank] for s in range(self.size)], dim=0).clone()
        self.sh.barrier.wait()
        return out

    @staticmethod
    def run(size: int, fn, *args_per_rank):
        """Run fn(comm, *args_per_rank[r]) for every rank r in its own thread; results by rank."""
        comms = ThreadComm.group(size)
        res, err = [None] * size, []

        def body(r):
            try:
                dev = torch.cuda.current_device() if torch.cuda.is_available() else None
                if dev is not None:
                    with torch.cuda.stream(torch.cuda.Stream(dev)):
                        res[r] = fn(comms[r], *[a[r] for a in args_per_rank])
                        torch.cuda.current_stream().synchronize()
                    cks.release_thread_contexts()
                else:
                    res[r] = fn(comms[r], *[a[r] for a in args_per_rank])
            except BaseException as e:          # unblock the others, re-raise below
                err.append(e)
                comms[r].sh.barrier.abort()

        th = [threading.Thread(target=body, args=(r,)) for r in range(size)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if err:
            raise err[0]
        return res


# ---- per-shard steps -------------------------------------------------------------------------

class CudaOps:
    """The per-shard steps as libcks kernels (the product path; no CPU fallback)."""
    occupancy = staticmethod(cks.occupancy)
    occupancy_sample = staticmethod(cks.occupancy_sample)
    occupancy_mask = staticmethod(cks.occupancy_mask)
    compress = staticmethod(cks.compress)
    compress_marking = staticmethod(cks.compress_marking)
    marks_occupancy = staticmethod(cks.marks_occupancy)
    partition = staticmethod(cks.partition)
    partition_count = staticmethod(cks.partition_count)
    partition_send = staticmethod(cks.partition_send)
    repack = staticmethod(cks.repack)
    sort_prefix = staticmethod(cks.sort_prefix)

    @staticmethod
    def sort(planes, bits, row_ids=None):
        return cks.sort(planes, bits, row_ids, want_sorted=True)

    @staticmethod
    def adjacent(sorted_planes, bits, sort_mask):
        return cks.adjacent_dbits(sorted_planes, bits, sort_mask, want_dbit=True)

    bulkload_block = staticmethod(cks.bulkload_block)
    bulkload_top = staticmethod(cks.bulkload_top)

    @staticmethod
    def first_build(keys, superset_kind):
        """One shard: the fused single first build (no tree: the sharded tree format follows)."""
        return cks.build(keys, superset_kind=superset_kind, tree=False)


# ---- host logic ----------------------------------------------------------------------------

def pick_splitters(samples: np.ndarray, size: int) -> np.ndarray:
    """G-1 splitters from the gathered regular samples (u32 rows: P plane words 0..np-1, then
    the row id), in the (P, row id) order: the samples at ranks i*S/G, i = 1..G-1."""
    s = np.asarray(samples, dtype=np.uint32).reshape(-1, samples.shape[-1])
    if size <= 1 or s.shape[0] == 0:
        return np.zeros((0, s.shape[1]), np.uint32)
    npl = s.shape[1] - 1
    order = np.lexsort([s[:, npl]] + [s[:, w] for w in range(npl)])   # last key primary: top plane
    srt = s[order]
    return np.ascontiguousarray(srt[[(i * srt.shape[0]) // size for i in range(1, size)]])


def regular_sample(count: int, per_rank: int) -> np.ndarray:
    """Positions of a regular sample of `per_rank` elements of a sorted shard of `count`."""
    s = min(per_rank, count)
    return ((2 * np.arange(s, dtype=np.int64) + 1) * count) // (2 * s) if s else np.zeros(0, np.int64)


def _height(n: int, per: int) -> int:
    """Levels of the bottom-up bulk load of n keys, per entries a node (0 for n = 0)."""
    h, c = 0, n
    while c > 0:
        c = (c + per - 1) // per
        h += 1
        if c == 1:
            break
    return h


def assemble_tree(outs: list[dict]) -> dict:
    """Host-side join of the distributed P:502 tree (every rank's out["tree"], rank order) into
    one node array set, levels concatenated leaves first (the layout of cks_bulkload):
    node_cnt [T], entry_rid / entry_child [T, fanout] (u32), entry_dbit [T, fanout] (u16)."""
    t0 = outs[0]["tree"]
    f, lstar = t0["fanout"], t0["lstar"]
    per = int(f * t0["fill"])
    subs = [o["tree"]["sub"] for o in outs]
    loc = [[int(s["shape"].level_nodes[l]) for l in range(lstar + 1)] if s is not None else [0] * (lstar + 1)
           for s in subs]
    top = t0["top"]
    top_lv = []
    c = sum(t0["children"])
    while c > 1:
        c = (c + per - 1) // per
        top_lv.append(c)
    lv = [sum(x[l] for x in loc) for l in range(lstar + 1)] + top_lv
    goff = np.cumsum([0] + lv)
    T = int(goff[-1])
    node_cnt = np.zeros(T, np.uint32)
    rid = np.full((T, f), 0xFFFFFFFF, np.uint32)
    child = np.full((T, f), 0xFFFFFFFF, np.uint32)
    edb = np.full((T, f), 0xFFFF, np.uint16)

    def host(t, a, b, dt):
        return t[a:b].cpu().numpy().view(dt)

    for l in range(lstar + 1):
        before = before_below = 0                        # this level's / the level below's nodes of earlier ranks
        for s, x in zip(subs, loc):
            if s is not None and x[l]:
                sh = s["shape"]
                lo, k = int(sh.level_offset[l]), x[l]
                g = int(goff[l]) + before
                node_cnt[g:g + k] = host(s["node_cnt"], lo, lo + k, np.uint32)
                rid[g:g + k] = host(s["entry_rid"], lo * f, (lo + k) * f, np.uint32).reshape(k, f)
                edb[g:g + k] = host(s["entry_dbit"], lo * f, (lo + k) * f, np.uint16).reshape(k, f)
                if l > 0:
                    io = lo - int(sh.level_nodes[0])
                    ch = host(s["entry_child"], io * f, (io + k) * f, np.uint32).reshape(k, f).astype(np.int64)
                    base = int(goff[l - 1]) + before_below - int(sh.level_offset[l - 1])
                    child[g:g + k] = np.where(ch != 0xFFFFFFFF, ch + base, 0xFFFFFFFF).astype(np.uint32)
            before += x[l]
            before_below += x[l - 1] if l > 0 else 0
    if top is not None:
        k = sum(top_lv)
        g = int(goff[lstar + 1])
        node_cnt[g:g + k] = host(top["node_cnt"], 0, k, np.uint32)
        rid[g:g + k] = host(top["entry_rid"], 0, k * f, np.uint32).reshape(k, f)
        edb[g:g + k] = host(top["entry_dbit"], 0, k * f, np.uint16).reshape(k, f)
        ch = host(top["entry_child"], 0, k * f, np.uint32).reshape(k, f).astype(np.int64)
        base = np.full((k, 1), g, np.int64)
        base[:top_lv[0]] = int(goff[lstar])              # the first top level indexes the child list
        child[g:g + k] = np.where(ch != 0xFFFFFFFF, ch + base, 0xFFFFFFFF).astype(np.uint32)
    return dict(height=len(lv), level_nodes=np.array(lv, np.uint64), node_cnt=node_cnt, entry_rid=rid,
                entry_child=child, entry_dbit=edb)


def _as_i32(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint32)).view(np.int32)


# ---- the sharded first build -------------------------------------------------------------------

def _exchange_fused(comm, ops, P, m, q, off, npl, dev):
    """The fused partition-and-send: the count pass, one all-gather of the
    G x G count matrix, receive buffers sized from its column, their addresses published, and
    ONE digit pass that writes every part straight into its receiver's buffer (peer device
    memory), then a barrier. Returns (received P planes, received row ids, send counts)."""
    G, r = comm.size, comm.rank
    n = int(P.shape[1])
    pc = ops.partition_count(P, m, q, G, off)
    cm = torch.stack(comm.allgather(pc)).cpu().numpy()          # cm[s][d]: elements s sends to d
    nr = int(cm[:, r].sum())
    # (one allocation per rank: its planes then its row ids, so one IPC handle serves both)
    buf = torch.empty((npl + 1) * max(nr, 1), dtype=torch.int32, device=dev)
    R = buf[:npl * nr].view(npl, nr)
    rids = buf[npl * max(nr, 1):npl * max(nr, 1) + nr]
    peers = comm.peer_tensors((buf,))
    dst_planes, dst_pitch, dst_rid = [], [], []
    for d in range(G):
        pb = peers[d][0]
        nd = int(cm[:, d].sum())
        at = int(cm[:r, d].sum())                                # this sender's start at receiver d
        dst_planes.append(pb.data_ptr() + 4 * at if npl else 0)
        dst_pitch.append(nd)
        dst_rid.append(pb.data_ptr() + 4 * (npl * max(nd, 1) + at))
    ops.partition_send(dst_planes, dst_pitch, dst_rid, dev.index)
    comm.barrier()                                               # every sender's stream has completed
    del peers
    return R, rids, [int(v) for v in cm[r]]


SPEC_MIN_KEYS = 1 << 20          # (as the single build, cks_api.cu kSpecMinKeys)
SPEC_SAMPLES = 65536             # rows over the whole column, split over the shards


def _all(comm, flag: bool, dev) -> bool:
    """Whether every rank's flag is set (one all-gather)."""
    if comm.size == 1:
        return bool(flag)
    return all(int(t.item()) for t in comm.allgather(torch.tensor([1 if flag else 0], dtype=torch.int64, device=dev)))


def build_sharded(keys: torch.Tensor, comm, ops=CudaOps, samples_per_rank: int = 256, fanout: int = 64,
                  fill: float = 1.0, tree: bool = True, superset_kind: int = cks.SUPERSET_BYTEOCC,
                  fused: bool | None = None) -> dict:
    """This rank's slice of the global first build. Returns dict(mask = exact D (same on all
    ranks), popcount, sort_mask = D+, sort_bits, perm = global row ids of the slice in order,
    dbit = D_i of the slice (against the global predecessor), packed = P_D of the slice,
    offset = global position of the slice's first key, n_total, send_counts, tree (rank 0))."""
    G, r = comm.size, comm.rank
    dev = keys.device
    n, B = int(keys.shape[0]), int(keys.shape[1])
    ns = [n] if G == 1 else [int(t.item()) for t in comm.allgather(torch.tensor([n], dtype=torch.int64, device=dev))]
    off, N = sum(ns[:r]), sum(ns)
    if N >= 1 << 32:
        raise ValueError("n_total >= 2^32 (u32 row ids)")
    if N == 0:
        e = torch.zeros(0, dtype=torch.int32, device=dev)
        z = np.zeros(B, np.uint8)
        return dict(mask=z, popcount=0, sort_mask=z, sort_bits=0, perm=e, dbit=e.to(torch.int16),
                    packed=torch.zeros((0, 0), dtype=torch.int32, device=dev), offset=0, n_total=0,
                    send_counts=[0] * G, tree=None)

    if G == 1 and hasattr(ops, "first_build"):
        # one shard, one part: the single first build (its mask from a row sample and the
        # compress marking the occupancy), then the sharded tree format
        fb = ops.first_build(keys, superset_kind)
        out = dict(mask=fb["mask"], popcount=fb["popcount"], sort_mask=fb["sort_mask"], sort_bits=fb["sort_bits"],
                   perm=fb["perm"], dbit=fb["dbit"], packed=fb["packed"], offset=0, n_total=N, send_counts=[n],
                   tree=None)
        if tree:
            out["tree"] = _slice_tree(comm, ops, out["perm"], out["dbit"], n, [n], fanout, fill, dev)
        return out

    # a1 + a3: D+ of the whole column from the union of the shard occupancies, and P_{D+}. Large
    # columns of 32/64-byte keys read the keys once for both (the speculative mask, DESIGN.md
    # Sec. 1.0): the union of strided row samples gives M' (inside D+), the compress by M' marks
    # every key's occupancy, and the union of those gives D+; the rare M' != D+ compresses again
    spec = (hasattr(ops, "compress_marking") and superset_kind == cks.SUPERSET_BYTEOCC and N >= SPEC_MIN_KEYS
            and B >= 32 and _all(comm, ops.marks_occupancy(keys) or n == 0, dev))   # (same answer on every rank)
    if spec:
        occ_s = ops.occupancy_sample(keys, max(1, SPEC_SAMPLES // G))
        Ms = ops.occupancy_mask(torch.stack(comm.allgather(occ_s)), N, superset_kind)
        P, occ = ops.compress_marking(keys, Ms)
        M = ops.occupancy_mask(torch.stack(comm.allgather(occ)), N, superset_kind)
        if not np.array_equal(M, Ms):
            P = ops.compress(keys, M)
        speculative = "held" if np.array_equal(M, Ms) else "retried"
    else:
        occ = ops.occupancy(keys)
        M = ops.occupancy_mask(occ[None] if G == 1 else torch.stack(comm.allgather(occ)), N, superset_kind)
        P = ops.compress(keys, M)
        speculative = None
    m = cks.popcount(M)
    npl = cks.nplanes(m)

    # splitters from a regular sample of every shard (none with one shard)
    q = None
    if G > 1:
        pos = torch.from_numpy(regular_sample(n, samples_per_rank)).to(dev)
        samp = torch.zeros((samples_per_rank, npl + 1), dtype=torch.int32, device=dev)
        if pos.numel():
            samp[:pos.numel(), :npl] = P[:, pos].t()
            samp[:pos.numel(), npl] = (pos + off).to(torch.int32)
        cnt = torch.tensor([pos.numel()], dtype=torch.int64, device=dev)
        counts = [int(c.item()) for c in comm.allgather(cnt)]
        rows = [t[:c].cpu().numpy().view(np.uint32) for t, c in zip(comm.allgather(samp), counts)]
        spl = pick_splitters(np.concatenate(rows) if rows else np.zeros((0, npl + 1), np.uint32), G)
        q = torch.from_numpy(_as_i32(spl)).to(dev).reshape(-1, npl + 1)

    # a5: stable partition, the one exchange, one stable sort on P
    if fused is None:
        fused = getattr(comm, "peer_access", False) and hasattr(ops, "partition_count") and keys.is_cuda
    if G == 1:                                                   # one part: the input order
        R, send_counts, rids = P, [n], None
    elif fused:
        R, rids, send_counts = _exchange_fused(comm, ops, P, m, q, off, npl, dev)
    else:
        Pp, ridp, pc = ops.partition(P, m, q, G, off)
        # the G x G count matrix in one collective: send counts (row r) and receive counts
        # (column r) without a second exchange
        cm = torch.stack(comm.allgather(pc)).cpu().numpy()
        send_counts = [int(v) for v in cm[r]]
        recv_counts = [int(v) for v in cm[:, r]]
        rids = comm.alltoallv(ridp, send_counts, recv_counts)    # per plane: no transposes
        R = torch.stack([comm.alltoallv(Pp[q], send_counts, recv_counts) for q in range(npl)]) if npl else \
            torch.zeros((0, rids.shape[0]), dtype=torch.int32, device=dev)
    nr = int(R.shape[1]) if rids is None else int(rids.shape[0])
    # sort by distinguishing prefixes (stable: the received order is the row-id order), D_i
    order, dbit, Dl, PDl = ops.sort_prefix(R, M, want_packed=True)
    if rids is None:                                             # one rank: row id = off + index
        perm = order + off if off else order
        ol = None
    else:
        ol = order.long()
        perm = rids[ol] if nr else rids                           # global row ids in (P, row id) order

    # a6 across the slice boundary: the previous non-empty slice's last key vs this first key
    Dl0 = Dl
    if G > 1:
        last = torch.zeros(npl + 1, dtype=torch.int32, device=dev)
        if nr:
            last[0] = 1
            last[1:] = R[:, ol[nr - 1]]
        lasts = comm.allgather(last)
        prev = next((lasts[k][1:] for k in range(r - 1, -1, -1) if int(lasts[k][0].item())), None)
        if prev is not None and nr:
            pair = torch.stack([prev, R[:, ol[0]]], dim=1).contiguous()
            Db, db = ops.adjacent(pair, m, M)
            dbit[0] = db[1]
            Dl = Dl | Db
        D = np.bitwise_or.reduce(np.stack([t.cpu().numpy() for t in comm.allgather(
            torch.from_numpy(np.ascontiguousarray(Dl)).to(dev))]), axis=0).astype(np.uint8)
    else:
        D = Dl

    # a7: P_D of the slice for the global D (the sort's own P_D when no other slice added bits)
    if PDl is not None and np.array_equal(D, Dl0):
        packed = PDl
    else:
        S2 = (R[:, ol].contiguous() if ol is not None else R[:, order.long()].contiguous()) if nr else R
        packed = ops.repack(S2, M, D) if not np.array_equal(D, M) else S2

    nrs = [nr] if G == 1 else [int(t.item()) for t in comm.allgather(torch.tensor([nr], dtype=torch.int64, device=dev))]
    out = dict(mask=D, popcount=cks.popcount(D), sort_mask=M, sort_bits=m, perm=perm, dbit=dbit, packed=packed,
               offset=sum(nrs[:r]), n_total=N, send_counts=send_counts, tree=None,
               speculative=speculative)

    # a8: a subtree per slice; the roots removed; the top layers over their children
    if tree and N:
        out["tree"] = _slice_tree(comm, ops, perm, dbit, nr, nrs, fanout, fill, dev)
    return out


def _slice_tree(comm, ops, perm, dbit, nr: int, nrs: list, fanout: int, fill: float, dev) -> dict:
    """this slice's subtree (levels 0..l*), its roots' children gathered, rank 0 builds the
    top layers over them."""
    G, r = comm.size, comm.rank
    per = int(fanout * fill)
    hs = [_height(nr, per)] if G == 1 else \
        [int(t.item()) for t in comm.allgather(torch.tensor([_height(nr, per)], dtype=torch.int64, device=dev))]
    hmin = min(h for h in hs if h > 0)
    lstar = max(0, hmin - 2)
    first_rank = next(k for k in range(G) if nrs[k] > 0)
    sub, cnt = None, 0
    if nr:
        sub = ops.bulkload_block(perm, dbit, fanout, fill, r == first_rank, lstar + 1)
        cnt = int(sub["shape"].level_nodes[lstar])
    span = per ** (lstar + 1)
    hi = torch.clamp(torch.arange(1, cnt + 1, device=dev, dtype=torch.int64) * span, max=nr) - 1
    cnts = [cnt] if G == 1 else \
        [int(t.item()) for t in comm.allgather(torch.tensor([cnt], dtype=torch.int64, device=dev))]
    pad = torch.zeros((max(1, max(cnts)), 2), dtype=torch.int32, device=dev)
    if cnt:
        pad[:cnt, 0] = perm[hi]
        pad[:cnt, 1] = sub["top_min"][:cnt].to(torch.int32)
    allc = [pad] if G == 1 else comm.allgather(pad)
    top = None
    if r == 0 and sum(cnts) > 1:
        crid = torch.cat([t[:c, 0] for t, c in zip(allc, cnts)]).contiguous()
        cmin = torch.cat([t[:c, 1] for t, c in zip(allc, cnts)]).to(torch.int16).contiguous()
        top = ops.bulkload_top(crid, cmin, fanout, fill)
    return dict(sub=sub, lstar=lstar, children=cnts, top=top, fanout=fanout, fill=fill, sizes=nrs)

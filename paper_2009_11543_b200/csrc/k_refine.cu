// k_refine.cu -- NEXT-1: first-build sort by distinguishing prefixes.
//
// The paper builds from compressed keys and notes that sorting needs only the bits that
// distinguish neighbours ("sort by distinguishing prefixes"; Theorem 2).
// The first build here sorts on chunks of the superset-compressed key P_M, most significant
// first:
//   round 0  LSD-sort all keys by the top T <= 64 bits (k_lsd.cu; T from a sample), carrying
//            that chunk + row id (and all of P_M when it has three planes);
//   round r  the keys whose prefix ties with a neighbour ("runs") are finished by comparing
//            their remaining bits when the run is short (k_ref_reg in registers after round 0
//            with P_M carried; k_ref_local / k_ref_warp / k_ref_cta from the compacted list),
//            and the long runs are re-sorted by (run, next 64 bits): one CTA per run when
//            every run fits (k_ref_cta_chunk), else a compact list (chunk of P_M by row id,
//            run index) LSD-sorted by (run, chunk) -- stable, so ties keep row-id order --
//            and written back into their run's positions, contiguous in the global order.
// A pair of neighbours is separated in the first round whose chunk differs; its D-bit
// is the first differing bit of that chunk, mapped through the M-offset table
// (P:479): D_i = moff[64 r + clz64(chunk_i XOR chunk_{i-1})]. Pairs equal in every chunk
// are duplicates (D_i = none, reading R3). The union of the D_i is the exact D.
//
// Kernels: k_ref_adj (round adjacency: D_i, tie flags, D accumulation), k_ref_reg (round-0
// adjacency fused with the in-tile short runs), k_ref_count / k_ref_scan / k_ref_scatter
// (compaction of the tied runs into the next round's list), k_ref_local / k_ref_warp /
// k_ref_cta (short and medium runs), k_ref_keep, k_ref_cta_chunk, k_ref_gather (chunk r of
// the listed rows), k_ref_put (sorted row ids back into place), k_prefix_sample (T).
#include <stdlib.h>

#include <type_traits>

#include "cks_internal.h"

namespace cks {

namespace {
constexpr int kRefThreads = 256;
constexpr int kRefItems = 16;                    // elements per thread in the compaction
constexpr int kRefTile = kRefThreads * kRefItems;

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t lane) {
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    return x - v;
}
}  // namespace

// Round adjacency over a sorted list of nr chunks (lo may be NULL: single-plane chunk;
// seg NULL: one segment; pos NULL: element k sits at global position k). Only the chunk bits
// in cmask are compared (round 0 sorts by the top T <= 64 bits).
__global__ void __launch_bounds__(kRefThreads)
k_ref_adj(const uint32_t* __restrict__ lo, const uint32_t* __restrict__ hi, const uint32_t* __restrict__ seg,
          const uint32_t* __restrict__ pos, uint64_t nr, uint32_t cbase, const uint16_t* __restrict__ moff,
          uint32_t m, uint32_t nwords, uint16_t* __restrict__ dbit, uint8_t* __restrict__ tie,
          uint32_t* __restrict__ dacc, int round0, unsigned long long cmask) {
    extern __shared__ uint32_t s_dyn[];
    uint32_t* s_bm = s_dyn;                                          // [nwords]
    uint16_t* s_moff = reinterpret_cast<uint16_t*>(s_dyn + nwords);  // [m]
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x) s_bm[w] = 0;
    for (uint32_t t = threadIdx.x; t < m; t += blockDim.x) s_moff[t] = moff[t];
    __syncthreads();
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nr; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = pos ? pos[k] : k;
        uint8_t t = 0;
        if (k == 0) {
            if (round0) dbit[g] = CKS_NONE_INTERNAL;
        } else if (!seg || seg[k] == seg[k - 1]) {
            const unsigned long long x = (((unsigned long long)(hi[k] ^ hi[k - 1]) << 32) |
                                          (lo ? (unsigned long long)(lo[k] ^ lo[k - 1]) : 0ull)) & cmask;
            if (x) {
                const uint32_t d = s_moff[cbase + (uint32_t)__clzll((long long)x)];
                dbit[g] = (uint16_t)d;
                const uint32_t w = d >> 5, b = 0x80000000u >> (d & 31);
                if (!(s_bm[w] & b)) atomicOr(&s_bm[w], b);
            } else {
                t = 1;
                if (round0) dbit[g] = CKS_NONE_INTERNAL;
            }
        }
        // (segment starts of later rounds keep the D_i found in an earlier round)
        tie[k] = t;
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x)
        if (s_bm[w]) atomicOr(&dacc[w], s_bm[w]);
}

// Element k belongs to a tied run if it ties with its predecessor or its successor; it
// starts a run if it does not tie with its predecessor.

// Tiles of kRefTile elements; thread t of a tile owns the 16 contiguous elements [16t, 16t+16)
// and holds their flags as a 16-bit mask (one 16-byte load). Member bits M = T | T>>1 | next<<15
// (T: the thread's flags, next: the flag after them), run starts S = M & ~T. The count takes
// kCompactTiles tiles per CTA and issues all their loads first; the scatter one tile per CTA
// (cfg5: count 28.5 -> 17 us, scatter 57 -> 37 us against per-element flags staged in shared
// memory; four tiles per scatter CTA lost on the dense lists of cfg4).
constexpr int kCompactTiles = 4;
__device__ __forceinline__ uint32_t flag_mask16(const uint8_t* __restrict__ tie, uint64_t nr, uint64_t k) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (k + 16 <= nr && ((reinterpret_cast<uintptr_t>(tie) & 15) == 0)) {
        v = *reinterpret_cast<const uint4*>(tie + k);
    } else if (k < nr) {
        uint8_t* b = reinterpret_cast<uint8_t*>(&v);
        for (int j = 0; j < 16; j++) b[j] = k + j < nr ? tie[k + j] : 0;
    }
    auto m4 = [](uint32_t w) {                                   // bit j: byte j nonzero
        const uint32_t b = __vcmpne4(w, 0u) & 0x01010101u;
        return (b | b >> 7 | b >> 14 | b >> 21) & 0xFu;
    };
    return m4(v.x) | m4(v.y) << 4 | m4(v.z) << 8 | m4(v.w) << 12;
}
// the CTA's tiles: live bits (tile t0 + u exists and has a flag), every thread's member and
// start masks
template <int TPC>
__device__ __forceinline__ uint32_t tile_masks(const uint8_t* __restrict__ tie, uint64_t nr, uint64_t ntiles,
                                               uint64_t t0, const uint8_t* __restrict__ any,
                                               uint32_t (&M)[TPC], uint32_t (&S)[TPC]) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t live = 0;
#pragma unroll
    for (int u = 0; u < TPC; u++)
        if (t0 + u < ntiles && (!any || any[t0 + u])) live |= 1u << u;
    uint32_t T[TPC], nx[TPC];
#pragma unroll
    for (int u = 0; u < TPC; u++) {
        const uint64_t k = (t0 + u) * kRefTile + 16 * (uint64_t)threadIdx.x;
        T[u] = (live >> u & 1u) ? flag_mask16(tie, nr, k) : 0u;
        nx[u] = (live >> u & 1u) && lane == 31 && k + 16 < nr ? (tie[k + 16] != 0) : 0u;
    }
#pragma unroll
    for (int u = 0; u < TPC; u++) {
        const uint32_t nb = __shfl_down_sync(0xffffffffu, T[u] & 1u, 1);
        const uint32_t next = lane == 31 ? nx[u] : nb;
        M[u] = (T[u] | T[u] >> 1 | next << 15) & 0xFFFFu;
        S[u] = M[u] & ~T[u];
    }
    return live;
}

// per tile: (members, run starts); a tile without a flag (`any`: nor the next tile's first) is
// not read
__global__ void __launch_bounds__(kRefThreads)
k_ref_count(const uint8_t* __restrict__ tie, uint64_t nr, uint64_t ntiles, uint32_t* __restrict__ cnt,
            const uint8_t* __restrict__ any) {
    __shared__ uint32_t s_red[kCompactTiles][2][kRefThreads / 32];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t t0 = (uint64_t)blockIdx.x * kCompactTiles;
    uint32_t M[kCompactTiles], S[kCompactTiles];
    const uint32_t live = tile_masks(tie, nr, ntiles, t0, any, M, S);
#pragma unroll
    for (int u = 0; u < kCompactTiles; u++) {
        const uint32_t cm = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(M[u]));
        const uint32_t cs = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(S[u]));
        if (lane == 0) { s_red[u][0][warp] = cm; s_red[u][1][warp] = cs; }
    }
    __syncthreads();
    if (threadIdx.x < 2 * kCompactTiles) {
        const uint32_t u = threadIdx.x >> 1, c = threadIdx.x & 1;
        if (t0 + u < ntiles) {
            uint32_t s = 0;
            if (live >> u & 1u)
                for (int w = 0; w < kRefThreads / 32; w++) s += s_red[u][c][w];
            cnt[2 * (t0 + u) + c] = s;
        }
    }
}

// exclusive scan of the tile counts in place (one CTA); totals to tot[0..1]. Thread t scans a
// contiguous range of tiles: one pass summing it, one block scan of the sums, one pass writing
// the prefixes (the counts are L2-resident: a few L2 round trips instead of one per 1024 tiles
// with four barriers each)
__global__ void __launch_bounds__(1024)
k_ref_scan(uint32_t* __restrict__ cnt, uint32_t ntiles, uint32_t* __restrict__ tot) {
    __shared__ uint32_t s_w[2][32];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t per = (ntiles + 1023) / 1024;
    const uint32_t b0 = min(ntiles, threadIdx.x * per), b1 = min(ntiles, b0 + per);
    uint2* c2 = reinterpret_cast<uint2*>(cnt);
    uint32_t v[2] = {0, 0};
#pragma unroll 4
    for (uint32_t b = b0; b < b1; b++) {
        const uint2 x = c2[b];
        v[0] += x.x;
        v[1] += x.y;
    }
    uint32_t e[2];
    for (int c = 0; c < 2; c++) {
        e[c] = warp_excl_scan(v[c], lane);
        if (lane == 31) s_w[c][warp] = e[c] + v[c];
    }
    __syncthreads();
    if (warp == 0) {
        for (int c = 0; c < 2; c++) {
            const uint32_t x = s_w[c][lane];
            const uint32_t ex = warp_excl_scan(x, lane);
            __syncwarp();
            s_w[c][lane] = ex;
            if (lane == 31) tot[c] = ex + x;
        }
    }
    __syncthreads();
    uint32_t r0 = s_w[0][warp] + e[0], r1 = s_w[1][warp] + e[1];
#pragma unroll 4
    for (uint32_t b = b0; b < b1; b++) {
        const uint2 x = c2[b];
        c2[b] = make_uint2(r0, r1);
        r0 += x.x;
        r1 += x.y;
    }
}

// write the next round's list: global position and run index of every tied element (and the
// list index of every run's first element), in element order: the warp walks its 512 elements
// 32 at a time (group i: threads 2i and 2i+1's masks, one shuffle each), skipping groups
// without a member, and places them by ballot prefix (coalesced stores)
template <int TPC>
__global__ void __launch_bounds__(kRefThreads)
k_ref_scatter(const uint8_t* __restrict__ tie, uint64_t nr, uint64_t ntiles, const uint32_t* __restrict__ pos,
              const uint32_t* __restrict__ cnt, uint32_t* __restrict__ pos_next, uint32_t* __restrict__ seg_next,
              uint32_t* __restrict__ run_off, uint32_t* __restrict__ run_pos, const uint8_t* __restrict__ any) {
    __shared__ uint32_t s_w[TPC][2][kRefThreads / 32];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ltm = (1u << lane) - 1u;
    const uint64_t t0 = (uint64_t)blockIdx.x * TPC;
    uint32_t M[TPC], S[TPC];
    const uint32_t live = tile_masks(tie, nr, ntiles, t0, any, M, S);
#pragma unroll
    for (int u = 0; u < TPC; u++) {
        const uint32_t cm = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(M[u]));
        const uint32_t cs = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(S[u]));
        if (lane == 0) { s_w[u][0][warp] = cm; s_w[u][1][warp] = cs; }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < TPC; u++) {
        const uint32_t nzb = __ballot_sync(0xffffffffu, M[u] != 0u);
        if (!(live >> u & 1u) || !nzb) continue;                 // (warp-uniform)
        const uint64_t tile = t0 + u;
        uint32_t om = cnt[2 * tile], os = cnt[2 * tile + 1];
        for (uint32_t w = 0; w < warp; w++) { om += s_w[u][0][w]; os += s_w[u][1][w]; }
        const uint64_t k0 = tile * kRefTile + warp * 32u * kRefItems + lane;
        auto put = [&](bool mb, bool st, uint32_t pk) {
            const uint32_t bm = __ballot_sync(0xffffffffu, mb), bs = __ballot_sync(0xffffffffu, st);
            if (mb) {
                const uint32_t o = om + __popc(bm & ltm);
                const uint32_t sg = os + __popc(bs & (ltm | (1u << lane))) - 1;   // runs started so far
                pos_next[o] = pk;
                seg_next[o] = sg;
                if (st && run_off) {
                    run_off[sg] = o;
                    run_pos[sg] = pk;                                 // position of the run's first key
                }
            }
            om += __popc(bm);
            os += __popc(bs);
        };
        // the groups holding a member
        uint32_t gz = 0;
#pragma unroll
        for (int i = 0; i < kRefItems; i++) gz |= (nzb >> (2 * i) & 3u) ? 1u << i : 0u;
        while (gz) {
            const int i = __ffs(gz) - 1;
            gz &= gz - 1u;
            const uint32_t src = 2u * i + (lane >> 4);
            const uint32_t mm = __shfl_sync(0xffffffffu, M[u], src), ss = __shfl_sync(0xffffffffu, S[u], src);
            const bool mb = mm >> (lane & 15) & 1u;
            const uint64_t k = k0 + 32 * i;
            put(mb, ss >> (lane & 15) & 1u, pos && mb ? pos[k] : (uint32_t)k);
        }
    }
}

// 64 bits of P_M starting at bit o (counted from its most significant bit; left-aligned planes)
// of the listed rows -- hi = bits [o, o+32), lo = bits [o+32, o+64) -- plus run and row id
__device__ __forceinline__ uint32_t pm_bits32(const uint32_t* pm, uint64_t pitch, uint32_t np, uint32_t o,
                                              uint32_t row) {
    const int q = (int)np - 1 - (int)(o >> 5);
    const uint32_t sh = o & 31;
    const uint32_t a = q >= 0 ? __ldg(pm + (uint64_t)q * pitch + row) : 0u;
    const uint32_t b = (sh && q >= 1) ? __ldg(pm + (uint64_t)(q - 1) * pitch + row) : 0u;
    return sh ? __funnelshift_l(b, a, sh) : a;
}

__global__ void __launch_bounds__(kRefThreads)
k_ref_gather(const uint32_t* __restrict__ pm, uint64_t pitch, uint32_t np, uint32_t o, const uint32_t* __restrict__ pos,
             const uint32_t* __restrict__ seg, const uint32_t* __restrict__ perm, uint64_t nr,
             uint32_t* __restrict__ out, uint64_t opitch, uint32_t* __restrict__ orid) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nr; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t row = perm[pos[k]];
        out[k] = pm_bits32(pm, pitch, np, o + 32, row);
        out[opitch + k] = pm_bits32(pm, pitch, np, o, row);
        out[2 * opitch + k] = seg[k];
        orid[k] = row;
    }
}

// Finish tied runs in place. Every element's "remaining key" is its P_M words from plane qtop
// down to 0 (the plane holding the first bit after the tied prefix; word qtop masked by fmask)
// -- read from the carried sorted planes at the run's positions when P_M is carried, else
// from P_M by row id -- and the run is sorted by (remaining key, row id): the stable order,
// a total order. D_i of each new neighbour pair = first differing remaining bit.
// By run length L:   L <= 4      k_ref_local, one thread, a 5-comparator network in registers
//                                (P_M read by row and more than 4 planes left: insertion sort on
//                                row ids with lazily read words, up to 16 keys);
//                    L <= 32     k_ref_warp, one warp, bitonic network over shuffles;
//                    L <= 2048   k_ref_cta, one CTA, bitonic sort in shared memory;
//                    longer      next LSD round (`done` = 0).
constexpr uint32_t kLocal = 4;
constexpr uint32_t kWarpRun = 32;
constexpr uint32_t kLazyRun = 16;                // pm path with more planes than registers
constexpr int kRegWords = 4;                     // remaining words held in registers (thread / warp paths)
constexpr uint32_t kCta = 2048;                  // medium runs: one CTA, bitonic sort in shared memory
constexpr uint32_t kCtaWords = 8;                // ... if at most this many P_M planes remain (measured:
                                                 // with 10 remaining planes, cfg4, gathering them by row
                                                 // id costs more than leaving the runs to the LSD round)

struct RunCtx {                                  // what every run finisher needs
    const uint32_t* pm;
    uint64_t pitch;
    uint32_t np;
    int qtop;
    uint32_t fmask;
    const uint16_t* moff;
    uint32_t* perm;
    uint16_t* dbit;
    uint32_t* carried;
};

// remaining word c (0 = plane qtop) of the element at global position p with row id `row`
__device__ __forceinline__ uint32_t rem_word(const RunCtx& R, int c, uint32_t p, uint32_t row) {
    const int q = R.qtop - c;
    const uint32_t v = R.carried ? R.carried[(uint64_t)q * R.pitch + p] : __ldg(R.pm + (uint64_t)q * R.pitch + row);
    return c == 0 ? v & R.fmask : v;
}
// write back element (words w, row id) to position p; D_i against the previous element's words
template <int W>
__device__ __forceinline__ void put_elem(const RunCtx& R, uint32_t p, const uint32_t (&w)[W], uint32_t row,
                                         const uint32_t* prev, uint32_t* s_bm) {
    CKS_DCHECK(p < R.pitch && row < R.pitch);
    R.perm[p] = row;
    if (R.carried)                                   // the carried planes follow their rows
        for (int c = 0; c <= R.qtop && c < W; c++) {
            const uint64_t at = (uint64_t)(R.qtop - c) * R.pitch + p;
            R.carried[at] = c == 0 ? (R.carried[at] & ~R.fmask) | w[0] : w[c];
        }
    if (!prev) return;
#pragma unroll
    for (int c = 0; c < W; c++) {
        const uint32_t x = w[c] ^ prev[c];
        if (x) {
            const uint32_t d = R.moff[32u * (R.np - 1 - (uint32_t)(R.qtop - c)) + (uint32_t)__clz(x)];
            R.dbit[p] = (uint16_t)d;
            const uint32_t b = 0x80000000u >> (d & 31);
            if (!(s_bm[d >> 5] & b)) atomicOr(&s_bm[d >> 5], b);
            return;
        }
    }
}

template <int W>
__device__ __forceinline__ bool key_less(const uint32_t (&a)[W], uint32_t ra, const uint32_t (&b)[W], uint32_t rb) {
#pragma unroll
    for (int c = 0; c < W; c++)
        if (a[c] != b[c]) return a[c] < b[c];
    return ra < rb;
}

// Positions handled per CTA / per thread by the round-0 finisher (k_ref_reg).
constexpr int kTileKeys = 2048;
constexpr int kTileItems = kTileKeys / kRefThreads;     // consecutive positions per thread (8)

// 8 consecutive u32 (positions p0..p0+7, p0 % 8 == 0) -- two 16-byte accesses when the whole
// group is in range and `vec` (16-byte aligned arrays), else element by element
__device__ __forceinline__ void ld8(const uint32_t* a, uint64_t p0, uint64_t n, bool vec, uint32_t (&v)[kTileItems]) {
    if (vec && p0 + kTileItems <= n) {
        const uint4 x = *reinterpret_cast<const uint4*>(a + p0), y = *reinterpret_cast<const uint4*>(a + p0 + 4);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
    } else {
#pragma unroll
        for (int j = 0; j < kTileItems; j++) v[j] = p0 + j < n ? a[p0 + j] : 0u;
    }
}
__device__ __forceinline__ void st8(uint32_t* a, uint64_t p0, uint64_t n, bool vec, const uint32_t (&v)[kTileItems]) {
    if (vec && p0 + kTileItems <= n) {
        *reinterpret_cast<uint4*>(a + p0) = make_uint4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<uint4*>(a + p0 + 4) = make_uint4(v[4], v[5], v[6], v[7]);
    } else {
#pragma unroll
        for (int j = 0; j < kTileItems; j++)
            if (p0 + j < n) a[p0 + j] = v[j];
    }
}

// Round-0 adjacency fused with finishing the short runs one thread holds (registers only; it
// replaces a shared-memory tile kernel with block scans and a member list, 0.65 -> 0.48 ms on
// cfg5 -- DESIGN.md Sec. 6.2). Thread = 8 consecutive
// sorted positions, CTA = 2048:
//   1. tie flag of every position against its predecessor on the top T bits, D_i of the others
//      (moff of the first differing P_M bit);
//   2. tied runs that lie inside the thread's 8 positions are sorted in registers by (remaining
//      P_M words, row id) -- the stable order -- with an odd-even transposition network whose
//      comparator (j, j+1) is enabled only when j+1 ties with j inside such a run;
//   3. runs of exactly two keys across two neighbouring lanes take one compare-exchange over
//      shuffles;
//   4. the members' D_i (first differing remaining bit, none for equal keys) are written and
//      their tie flags cleared. Runs crossing a thread boundary with 3+ keys, or a warp
//      boundary, keep their tie flags for the compaction that follows (round 1: k_ref_local /
//      k_ref_warp / k_ref_cta), as do runs longer than a thread.
// Remaining key of a position (WC = qtop + 1 words, planes qtop .. 0 of the carried sorted P_M,
// word 0 masked by fmask): WC 1: k = w0; WC 2: k = w0:w1; WC 3: k = w0:w1, x = w2.
// Strict order of remaining keys. The row id is not compared: round 0 is a stable LSD sort of
// the rows in input order (implicit, increasing row ids), so a tied run enters the networks in
// increasing row-id order, and a transposition network that swaps only on "strictly less"
// keeps equal keys in that order -- the (key, row id) order without comparing row ids.
template <int WC>
__device__ __forceinline__ bool rk_less(unsigned long long ka, uint32_t xa, unsigned long long kb, uint32_t xb) {
    if (WC == 3) return ka < kb || (ka == kb && xa < xb);
    return ka < kb;
}

template <int WC, int NP>
__global__ void __launch_bounds__(kRefThreads, 3)
k_ref_reg(RunCtx R, const uint32_t* __restrict__ lo, const uint32_t* __restrict__ hi, uint64_t n,
          unsigned long long cmask, bool vec, uint8_t* __restrict__ tie, uint32_t* __restrict__ dacc,
          uint32_t* __restrict__ handled, uint8_t* __restrict__ any) {
    static_assert(WC >= 1 && WC <= 3 && (NP == 3 || NP == 4) && WC <= NP, "carried remaining words");
    constexpr int I = kTileItems;                                 // 8 positions per thread
    // D of the CTA as a byte per P_M bit index (a plain byte store marks a bit: every writer
    // stores 1, so the races are benign and no variable 64-bit shift is needed)
    __shared__ uint8_t s_dm[32 * NP];
    __shared__ uint32_t s_cnt;
    for (uint32_t t = threadIdx.x; t < 32u * NP; t += blockDim.x) s_dm[t] = 0;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    // persistent CTAs: D and the counts are reduced once per CTA, not per tile (one global atomic
    // per D-bit per CTA)
    uint32_t hm = 0;
    const uint64_t ntiles = (n + kTileKeys - 1) / kTileKeys;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t p0 = (tile * kRefThreads + threadIdx.x) * I;
        auto top = [&](uint64_t k) -> unsigned long long {
            return (((unsigned long long)__ldg(hi + k) << 32) | (unsigned long long)__ldg(lo + k)) & cmask;
        };
        // A. loads: chunk words (hi = plane NP-1, lo = plane NP-2 of the carried planes), row
        // ids, the planes below the chunk (0, and 1 when NP = 4)
        uint32_t vh[I], vl[I], vr[I], v0[I], v1[I];
        ld8(hi, p0, n, vec, vh);
        ld8(lo, p0, n, vec, vl);
        ld8(R.perm, p0, n, vec, vr);
        ld8(R.carried, p0, n, vec, v0);                               // plane 0
        if (NP == 4) ld8(R.carried + R.pitch, p0, n, vec, v1);        // plane 1
        else {
#pragma unroll
            for (int j = 0; j < I; j++) v1[j] = 0u;
        }
        const uint32_t vm = p0 >= n ? 0u : (p0 + I <= n ? 0xFFu : (1u << (uint32_t)(n - p0)) - 1u);
        unsigned long long tk[I];
    #pragma unroll
        for (int j = 0; j < I; j++) tk[j] = (((unsigned long long)vh[j] << 32) | vl[j]) & cmask;
        // neighbours across the thread: the previous position's top bits, the next's tie
        unsigned long long tprev = __shfl_up_sync(0xffffffffu, tk[I - 1], 1);
        if (lane == 0 && p0 > 0 && p0 - 1 < n) tprev = top(p0 - 1);
        // B. tie bits (position j ties with j-1) and D_i of the others from the top T bits
        uint32_t tb = 0;
        uint16_t odb[I];
    #pragma unroll
        for (int j = 0; j < I; j++) {
            const unsigned long long pv = j ? tk[j - 1] : tprev;
            odb[j] = CKS_NONE_INTERNAL;
            if ((vm >> j & 1) && p0 + j > 0) {
                const unsigned long long x = tk[j] ^ pv;
                if (x) {
                    const uint32_t pmb = (uint32_t)__clzll((long long)x);   // < T <= 64
                    odb[j] = __ldg(R.moff + pmb);
                    s_dm[pmb] = 1;
                } else {
                    tb |= 1u << j;
                }
            }
        }
        const uint32_t tbn = __shfl_down_sync(0xffffffffu, tb, 1);      // next lane's tie bits
        bool tie_next = lane < 31 ? (tbn & 1u) != 0 : false;
        if (lane == 31 && (vm >> (I - 1) & 1) && p0 + I < n) tie_next = top(p0 + I) == tk[I - 1];
        // C. runs inside the thread: links L (bit j: j ties with j-1, j >= 1); runs open to the left
        // (position 0 ties with the previous lane) or right (the next lane's first position ties
        // with position 7) are not finished here
        const uint32_t L = tb & 0xFEu;
        uint32_t hl = L;
        if (tb & 1u) {                                                // run through position 0
            const uint32_t e = (uint32_t)__ffs(~(L | 1u)) - 1u;       // first position after it
            hl &= ~(((1u << e) - 1u) & ~1u);
        }
        if (tie_next) {                                               // run through position 7
            const uint32_t s = 31u - (uint32_t)__clz(~L & 0xFFu);     // its first position
            hl &= ~(0xFFu & ~((2u << s) - 1u));
        }
        // remaining keys (plane q of position j, q compile-time: NP-1 -> vh, NP-2 -> vl, 1 -> v1, 0 -> v0)
    #define CKS_PV(q, j) ((q) == NP - 1 ? vh[j] : (q) == NP - 2 ? vl[j] : (q) == 1 ? v1[j] : v0[j])
    #define CKS_PV2(q, j) ((q) == NP - 1 ? vh[j] : (q) == NP - 2 ? vl[j] : (q) == 1 ? v1[j] : v0[j])
        unsigned long long key[I];
        uint32_t kx[I], topw[I];                                      // topw: word 0's chunk bits (equal in a run)
    #pragma unroll
        for (int j = 0; j < I; j++) {
            const uint32_t w = CKS_PV(WC - 1, j);                     // plane qtop = WC - 1
            topw[j] = w & ~R.fmask;
            const uint32_t w0 = w & R.fmask;
            if (WC == 1) key[j] = w0;
            else key[j] = ((unsigned long long)w0 << 32) | CKS_PV(WC - 2, j);
    #undef CKS_PV
            kx[j] = WC == 3 ? CKS_PV2(0, j) : 0u;
        }
    #undef CKS_PV2
        // D. odd-even transposition network over the handled runs: L phases sort runs of up to L
        // keys, so the warp runs as many phases as its longest handled run (mostly 2-4), each
        // comparator a branch-free select
        bool changed = false;
        uint32_t runmax = 0;                                          // longest handled run (keys)
        {
            uint32_t h = hl, len = 1;
    #pragma unroll
            for (int j = 1; j < I; j++) {
                len = (h >> j & 1u) ? len + 1 : 1u;
                runmax = len > runmax ? len : runmax;
            }
            if (!hl) runmax = 0;
        }
        const uint32_t phases = __reduce_max_sync(0xffffffffu, runmax);
        auto cex = [&](int j) {
            const bool sw = (hl >> (j + 1) & 1u) && rk_less<WC>(key[j + 1], kx[j + 1], key[j], kx[j]);
            const unsigned long long ka = key[j], kb = key[j + 1];
            key[j] = sw ? kb : ka;
            key[j + 1] = sw ? ka : kb;
            if (WC == 3) {
                const uint32_t xa = kx[j], xb = kx[j + 1];
                kx[j] = sw ? xb : xa;
                kx[j + 1] = sw ? xa : xb;
            }
            const uint32_t ra = vr[j], rb = vr[j + 1];
            vr[j] = sw ? rb : ra;
            vr[j + 1] = sw ? ra : rb;
            changed |= sw;
        };
        for (uint32_t ph = 0; ph < phases; ph += 2) {
    #pragma unroll
            for (int j = 0; j + 1 < I; j += 2) cex(j);
            if (ph + 1 < phases) {
    #pragma unroll
                for (int j = 1; j + 1 < I; j += 2) cex(j);
            }
        }
        // E. D_i of the handled runs' members after their first
    #pragma unroll
        for (int j = 1; j < I; j++) {
            if (hl >> j & 1u) {
                const unsigned long long x = key[j] ^ key[j - 1];
                const uint32_t b0 = 32u * (R.np - (uint32_t)WC);
                int fd = -1;
                if (x) fd = (int)(b0 + (uint32_t)__clzll((long long)x) - (WC == 1 ? 32u : 0u));
                else if (WC == 3 && (kx[j] ^ kx[j - 1])) fd = (int)(b0 + 64u + (uint32_t)__clz(kx[j] ^ kx[j - 1]));
                odb[j] = CKS_NONE_INTERNAL;
                if (fd >= 0) {
                    odb[j] = __ldg(R.moff + fd);
                    s_dm[fd] = 1;
                }
            }
        }
        // E2. runs across two lanes: a second network over the window [4, 12) of lane t (its
        // positions 4..7 and lane t+1's 0..3), for the run holding window positions 3 and 4 when
        // it lies inside the window (runs of up to 5 keys always do); not across warps
        const uint32_t wl = ((tb >> 4) | (tbn << 4)) & 0xFFu;       // bit i: window i ties with i-1
        uint32_t hl2 = 0;
        if (lane < 31 && (wl >> 4 & 1u) && (wl & 0x0Fu) != 0x0Fu) {
            const uint32_t a = 31u - (uint32_t)__clz(~wl & 0x0Fu);       // the run's first window position
            const uint32_t hz = ~wl & 0xE0u;
            const uint32_t e = hz ? (uint32_t)__ffs(hz) - 1u : 8u;       // first window position after it
            if (e < 8u || !(tbn >> 4 & 1u)) hl2 = ((1u << e) - 1u) & ~((2u << a) - 1u);
        }
        // the window's positions 0..3 are key[4..7] (in place); 4..7 the next lane's 0..3 (nk)
        unsigned long long nk[4];
        uint32_t nx[4], nr[4];
        uint16_t nd[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            nk[j] = __shfl_down_sync(0xffffffffu, key[j], 1);
            nx[j] = WC == 3 ? __shfl_down_sync(0xffffffffu, kx[j], 1) : 0u;
            nr[j] = __shfl_down_sync(0xffffffffu, vr[j], 1);
            nd[j] = (uint16_t)__shfl_down_sync(0xffffffffu, (uint32_t)odb[j], 1);
        }
#define CKS_WK(j) (*((j) < 4 ? &key[4 + (j)] : &nk[(j) - 4]))
#define CKS_WX(j) (*((j) < 4 ? &kx[4 + (j)] : &nx[(j) - 4]))
#define CKS_WR(j) (*((j) < 4 ? &vr[4 + (j)] : &nr[(j) - 4]))
#define CKS_WD(j) (*((j) < 4 ? &odb[4 + (j)] : &nd[(j) - 4]))
        const uint32_t phases2 = __reduce_max_sync(0xffffffffu, hl2 ? (uint32_t)__popc(hl2) + 1u : 0u);
        bool wchanged = false;
        auto wcex = [&](auto jc) {
            constexpr int j = decltype(jc)::value;
            const bool sw = (hl2 >> (j + 1) & 1u) &&
                            rk_less<WC>(CKS_WK(j + 1), CKS_WX(j + 1), CKS_WK(j), CKS_WX(j));
            const unsigned long long ka = CKS_WK(j), kb = CKS_WK(j + 1);
            CKS_WK(j) = sw ? kb : ka;
            CKS_WK(j + 1) = sw ? ka : kb;
            if (WC == 3) {
                const uint32_t xa = CKS_WX(j), xb = CKS_WX(j + 1);
                CKS_WX(j) = sw ? xb : xa;
                CKS_WX(j + 1) = sw ? xa : xb;
            }
            const uint32_t ra = CKS_WR(j), rb = CKS_WR(j + 1);
            CKS_WR(j) = sw ? rb : ra;
            CKS_WR(j + 1) = sw ? ra : rb;
            wchanged |= sw;
        };
        using I0 = std::integral_constant<int, 0>;
        using I1 = std::integral_constant<int, 1>;
        using I2 = std::integral_constant<int, 2>;
        using I3 = std::integral_constant<int, 3>;
        using I4 = std::integral_constant<int, 4>;
        using I5 = std::integral_constant<int, 5>;
        using I6 = std::integral_constant<int, 6>;
        for (uint32_t ph = 0; ph < phases2; ph += 2) {
            wcex(I0{}); wcex(I2{}); wcex(I4{}); wcex(I6{});
            if (ph + 1 < phases2) { wcex(I1{}); wcex(I3{}); wcex(I5{}); }
        }
        auto wdi = [&](auto jc) {
            constexpr int j = decltype(jc)::value;
            if (hl2 >> j & 1u) {
                const unsigned long long x = CKS_WK(j) ^ CKS_WK(j - 1);
                const uint32_t b0 = 32u * (R.np - (uint32_t)WC);
                int fd = -1;
                if (x) fd = (int)(b0 + (uint32_t)__clzll((long long)x) - (WC == 1 ? 32u : 0u));
                else if (WC == 3 && (CKS_WX(j) ^ CKS_WX(j - 1)))
                    fd = (int)(b0 + 64u + (uint32_t)__clz(CKS_WX(j) ^ CKS_WX(j - 1)));
                CKS_WD(j) = CKS_NONE_INTERNAL;
                if (fd >= 0) {
                    CKS_WD(j) = __ldg(R.moff + fd);
                    s_dm[fd] = 1;
                }
            }
        };
        wdi(I1{}); wdi(I2{}); wdi(I3{}); wdi(I4{}); wdi(I5{}); wdi(I6{}); wdi(std::integral_constant<int, 7>{});
#undef CKS_WK
#undef CKS_WX
#undef CKS_WR
#undef CKS_WD
        changed |= wchanged;                                      // (the run always holds window position 3)
        const uint32_t hl2p = __shfl_up_sync(0xffffffffu, hl2, 1);   // the previous lane's window
        const bool chp = __shfl_up_sync(0xffffffffu, (uint32_t)wchanged, 1) != 0u;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const unsigned long long k2 = __shfl_up_sync(0xffffffffu, nk[j], 1);
            const uint32_t x2 = WC == 3 ? __shfl_up_sync(0xffffffffu, nx[j], 1) : 0u;
            const uint32_t r2 = __shfl_up_sync(0xffffffffu, nr[j], 1);
            const uint16_t d2 = (uint16_t)__shfl_up_sync(0xffffffffu, (uint32_t)nd[j], 1);
            if (lane > 0 && hl2p) { key[j] = k2; kx[j] = x2; vr[j] = r2; odb[j] = d2; }
        }
        if (lane > 0 && hl2p && chp) changed = true;
        // F. write back: tie flags of the unfinished runs only, D_i, and the reordered groups
        const uint32_t tout = tb & ~hl & ~((hl2 & 0x0Eu) << 4) & ~(lane > 0 ? (hl2p >> 4) & 0x0Fu : 0u);
        if (changed) {
            st8(R.perm, p0, n, vec, vr);
            uint32_t ow[I];
    #pragma unroll
            for (int c = 0; c < WC; c++) {
                const int q = WC - 1 - c;                                 // plane of remaining word c
    #pragma unroll
                for (int j = 0; j < I; j++) {
                    (void)q;
                    if (c == 0) ow[j] = topw[j] | (uint32_t)(WC == 1 ? key[j] : key[j] >> 32);
                    else if (c == 1) ow[j] = (uint32_t)key[j];
                    else ow[j] = kx[j];
                }
                st8(R.carried + (uint64_t)q * R.pitch, p0, n, vec, ow);
            }
        }
        uint32_t ot[2] = {0, 0};
    #pragma unroll
        for (int j = 0; j < I; j++) {
            ot[j >> 2] |= (tout >> j & 1u) << (8 * (j & 3));
            if (tout >> j & 1u) odb[j] = CKS_NONE_INTERNAL;
        }
        if (vec && p0 + I <= n) {
            *reinterpret_cast<uint2*>(tie + p0) = make_uint2(ot[0], ot[1]);
            *reinterpret_cast<uint4*>(R.dbit + p0) =
                make_uint4(odb[0] | ((uint32_t)odb[1] << 16), odb[2] | ((uint32_t)odb[3] << 16),
                           odb[4] | ((uint32_t)odb[5] << 16), odb[6] | ((uint32_t)odb[7] << 16));
        } else {
            for (int j = 0; j < I; j++)
                if (p0 + j < n) { tie[p0 + j] = (uint8_t)(tout >> j & 1u); R.dbit[p0 + j] = odb[j]; }
        }
        if (any && tout) {                                            // compaction tiles with ties left
            const uint64_t c = p0 / kRefTile;
            any[c] = 1;
            if ((tout & 1u) && c && p0 % kRefTile == 0) any[c - 1] = 1;
        }
        hm += (uint32_t)__popc(hl | (hl >> 1)) + (uint32_t)__popc(hl2 | (hl2 >> 1));
    }
    // G. counts and D
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) hm += __shfl_xor_sync(0xffffffffu, hm, o);
    if (lane == 0) atomicAdd(&s_cnt, hm);
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < 32u * NP; t += blockDim.x)
        if (s_dm[t]) {
            const uint32_t d = __ldg(R.moff + t);
            atomicOr(&dacc[d >> 5], 0x80000000u >> (d & 31));
        }
    if (threadIdx.x == 0 && s_cnt) atomicAdd(handled, s_cnt);
}

// Thread per run: short runs (<= 4, registers only: a fixed network, static indices); longer
// runs are routed to the warp list, the CTA list or the next LSD round.
__global__ void __launch_bounds__(kRefThreads)
k_ref_local(RunCtx R, const uint32_t* __restrict__ run_pos, const uint32_t* __restrict__ run_off, uint64_t nseg,
            uint64_t nn, uint32_t* __restrict__ dacc, uint8_t* __restrict__ done, uint32_t nwords,
            uint32_t* __restrict__ mlist, uint32_t* __restrict__ wlist, uint32_t* __restrict__ mcount,
            uint32_t cta_max) {
    constexpr int W = kRegWords;
    __shared__ uint32_t s_bm[kMaxBits / 32];                         // D bits found by this block
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x) s_bm[w] = 0;
    __syncthreads();
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t sweeps = (nseg + nthreads - 1) / nthreads;       // uniform trip count (block barrier below)
    const int Wr = R.qtop + 1;
    for (uint64_t it = 0; it < sweeps; it++) {
        const uint64_t s = it * nthreads + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (s >= nseg) continue;
        const uint32_t k0 = run_off[s];
        const uint32_t k1 = s + 1 < nseg ? run_off[s + 1] : (uint32_t)nn;
        const uint32_t L = k1 - k0;
        const uint32_t p0 = run_pos[s];                               // position of the run's first key
        uint8_t fin = 1;
        if (L <= kLocal && Wr <= W) {
            uint32_t r[4], w[4][W];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                r[j] = 0xFFFFFFFFu;                                  // padding sorts last
#pragma unroll
                for (int c = 0; c < W; c++) w[j][c] = 0xFFFFFFFFu;
                if ((uint32_t)j < L) {
                    r[j] = R.perm[p0 + j];
#pragma unroll
                    for (int c = 0; c < W; c++) w[j][c] = c < Wr ? rem_word(R, c, p0 + j, r[j]) : 0u;
                }
            }
            auto cswap = [&](int x, int y) {
                if (key_less<W>(w[y], r[y], w[x], r[x])) {
                    const uint32_t tr = r[x]; r[x] = r[y]; r[y] = tr;
#pragma unroll
                    for (int c = 0; c < W; c++) { const uint32_t tw = w[x][c]; w[x][c] = w[y][c]; w[y][c] = tw; }
                }
            };
            cswap(0, 1); cswap(2, 3); cswap(0, 2); cswap(1, 3); cswap(1, 2);
#pragma unroll
            for (int j = 0; j < 4; j++)
                if ((uint32_t)j < L) put_elem<W>(R, p0 + j, w[j], r[j], j ? w[j - 1] : nullptr, s_bm);
        } else if (L <= kLazyRun && !R.carried && (Wr > W || L <= kLocal)) {
            // more remaining planes than registers: an insertion sort on row ids with every
            // key's first remaining word loaded up front (L independent loads; most pairs
            // differ there) and the deeper words read from P_M by row only for ties in it
            auto deeper = [&](uint32_t a, uint32_t b, uint32_t* tt) -> int {
                for (int c = 1; c < Wr; c++) {
                    const uint32_t wa = rem_word(R, c, 0, a), wb = rem_word(R, c, 0, b);
                    if (wa != wb) {
                        if (tt) *tt = 32u * (R.np - 1 - (uint32_t)(R.qtop - c)) + (uint32_t)__clz(wa ^ wb);
                        return wa < wb ? -1 : 1;
                    }
                }
                return 0;
            };
            auto cmp = [&](uint32_t fa, uint32_t a, uint32_t fb, uint32_t b, uint32_t* tt) -> int {
                if (fa != fb) {
                    if (tt) *tt = 32u * (R.np - 1 - (uint32_t)R.qtop) + (uint32_t)__clz(fa ^ fb);
                    return fa < fb ? -1 : 1;
                }
                return deeper(a, b, tt);
            };
            uint32_t r[kLazyRun], f[kLazyRun];
            for (uint32_t j = 0; j < L; j++) r[j] = R.perm[p0 + j];
            for (uint32_t j = 0; j < L; j++) f[j] = rem_word(R, 0, 0, r[j]);
            for (uint32_t j = 1; j < L; j++) {
                const uint32_t x = r[j], fx = f[j];
                uint32_t i = j;
                while (i > 0) {
                    const int c = cmp(f[i - 1], r[i - 1], fx, x, nullptr);
                    if (c < 0 || (c == 0 && r[i - 1] < x)) break;
                    r[i] = r[i - 1];
                    f[i] = f[i - 1];
                    i--;
                }
                r[i] = x;
                f[i] = fx;
            }
            for (uint32_t j = 0; j < L; j++) {
                R.perm[p0 + j] = r[j];
                uint32_t tt = 0;
                if (j && cmp(f[j - 1], r[j - 1], f[j], r[j], &tt) != 0) {
                    const uint32_t d = R.moff[tt];
                    R.dbit[p0 + j] = (uint16_t)d;
                    const uint32_t b = 0x80000000u >> (d & 31);
                    if (!(s_bm[d >> 5] & b)) atomicOr(&s_bm[d >> 5], b);
                }
            }
        } else if (L <= kWarpRun && Wr <= W) {
            wlist[atomicAdd(mcount + 2, 1u)] = (uint32_t)s;
        } else if (L <= cta_max && Wr <= (int)kCtaWords) {
            mlist[atomicAdd(mcount, 1u)] = (uint32_t)s;
        } else {
            fin = 0;                                                 // long run: next round
            atomicAdd(mcount + 1, 1u);
            atomicMax(mcount + 3, L);
        }
        done[s] = fin;
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x)
        if (s_bm[w]) atomicOr(&dacc[w], s_bm[w]);
}

// Warp per run (5..32 keys): lane j holds element j (padding sorts last); bitonic network by
// shuffles; lane j writes the j-th smallest and its D_i against lane j-1's element.
__global__ void __launch_bounds__(kRefThreads)
k_ref_warp(RunCtx R, const uint32_t* __restrict__ run_pos, const uint32_t* __restrict__ run_off, uint64_t nseg,
           uint64_t nn, uint32_t* __restrict__ dacc, uint32_t nwords, const uint32_t* __restrict__ wlist,
           const uint32_t* __restrict__ mcount) {
    constexpr int W = kRegWords;
    __shared__ uint32_t s_bm[kMaxBits / 32];
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x) s_bm[w] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t cnt = mcount[2];
    const int Wr = R.qtop + 1;
    const uint32_t nwarps = gridDim.x * (blockDim.x / 32);
    for (uint32_t wi = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); wi < cnt; wi += nwarps) {
        const uint32_t s = wlist[wi];
        const uint32_t k0 = run_off[s];
        const uint32_t k1 = s + 1 < nseg ? run_off[s + 1] : (uint32_t)nn;
        const uint32_t L = k1 - k0;
        const uint32_t p0 = run_pos[s];
        uint32_t r = 0xFFFFFFFFu, w[W];
#pragma unroll
        for (int c = 0; c < W; c++) w[c] = 0xFFFFFFFFu;
        if (lane < L) {
            r = R.perm[p0 + lane];
#pragma unroll
            for (int c = 0; c < W; c++) w[c] = c < Wr ? rem_word(R, c, p0 + lane, r) : 0u;
        }
#pragma unroll
        for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                uint32_t ow[W];
#pragma unroll
                for (int c = 0; c < W; c++) ow[c] = __shfl_xor_sync(0xffffffffu, w[c], stride);
                const uint32_t orr = __shfl_xor_sync(0xffffffffu, r, stride);
                const bool lower = (lane & stride) == 0;             // this lane keeps the min if ascending
                const bool up = (lane & size) == 0;
                const bool other_less = key_less<W>(ow, orr, w, r);
                if (other_less == (lower == up)) {
                    r = orr;
#pragma unroll
                    for (int c = 0; c < W; c++) w[c] = ow[c];
                }
            }
        }
        uint32_t pw[W];
#pragma unroll
        for (int c = 0; c < W; c++) pw[c] = __shfl_up_sync(0xffffffffu, w[c], 1);
        if (lane < L) put_elem<W>(R, p0 + lane, w, r, lane ? pw : nullptr, s_bm);
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x)
        if (s_bm[w]) atomicOr(&dacc[w], s_bm[w]);
}

// Medium runs (kLocal < L <= kCta): one CTA per run (grid-stride over the list made by
// k_ref_local). The run's row ids and remaining P_M words (planes qtop .. 0, from the
// carried sorted planes or by row id) are staged in shared memory and an index array is
// bitonic-sorted by (words, row id) -- the stable order; then perm, the carried planes and
// the D_i (first differing remaining bit) are written at the run's positions.
__global__ void __launch_bounds__(kRefThreads)
k_ref_cta(const uint32_t* __restrict__ pm, uint64_t pitch, uint32_t np, int qtop, const uint16_t* __restrict__ moff,
          const uint32_t* __restrict__ run_pos, const uint32_t* __restrict__ run_off, uint64_t nseg, uint64_t nn,
          uint32_t* __restrict__ perm, uint16_t* __restrict__ dbit, uint32_t* __restrict__ dacc,
          uint32_t* __restrict__ carried, uint32_t nwords, const uint32_t* __restrict__ mlist,
          const uint32_t* __restrict__ mcount, uint32_t fmask) {
    extern __shared__ uint32_t s_dyn[];
    uint32_t* s_rid = s_dyn;                                         // [kCta]
    uint32_t* s_kw = s_rid + kCta;                                   // [Wr][kCta], word 0 = plane qtop
    uint16_t* s_idx = reinterpret_cast<uint16_t*>(s_kw + (qtop + 1) * kCta);   // [kCta]
    __shared__ uint32_t s_bm[kMaxBits / 32];
    const uint32_t Wr = (uint32_t)qtop + 1;
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x) s_bm[w] = 0;
    const uint32_t cnt = *mcount;
    for (uint32_t mi = blockIdx.x; mi < cnt; mi += gridDim.x) {
        const uint32_t s = mlist[mi];
        const uint32_t k0 = run_off[s];
        const uint32_t k1 = s + 1 < nseg ? run_off[s + 1] : (uint32_t)nn;
        const uint32_t L = k1 - k0;
        const uint32_t p0 = run_pos[s];
        uint32_t P2 = 1;
        while (P2 < L) P2 <<= 1;
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < L; j += blockDim.x) {
            const uint32_t row = perm[p0 + j];
            s_rid[j] = row;
            for (uint32_t q = 0; q < Wr; q++)
                s_kw[q * kCta + j] = (carried ? carried[(uint64_t)(qtop - (int)q) * pitch + p0 + j]
                                              : __ldg(pm + (uint64_t)(qtop - (int)q) * pitch + row)) &
                                     (q == 0 ? fmask : 0xFFFFFFFFu);
        }
        for (uint32_t j = threadIdx.x; j < P2; j += blockDim.x) s_idx[j] = (uint16_t)j;
        __syncthreads();
        auto less = [&](uint32_t a, uint32_t b) -> bool {            // padding (>= L) sorts last
            if (a >= L || b >= L) return a < b;
            for (uint32_t q = 0; q < Wr; q++) {
                const uint32_t x = s_kw[q * kCta + a], y = s_kw[q * kCta + b];
                if (x != y) return x < y;
            }
            return s_rid[a] < s_rid[b];
        };
        for (uint32_t size = 2; size <= P2; size <<= 1) {
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t i = threadIdx.x; i < P2 / 2; i += blockDim.x) {
                    const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    const uint32_t a = s_idx[lo], b = s_idx[hi];
                    if (less(b, a) == up) { s_idx[lo] = (uint16_t)b; s_idx[hi] = (uint16_t)a; }
                }
                __syncthreads();
            }
        }
        for (uint32_t j = threadIdx.x; j < L; j += blockDim.x) {
            const uint32_t a = s_idx[j];
            perm[p0 + j] = s_rid[a];
            if (carried) {                                      // reorder the carried planes too
                for (uint32_t q = 0; q < Wr; q++) {
                    const uint64_t at = (uint64_t)(qtop - (int)q) * pitch + p0 + j;
                    carried[at] = q == 0 ? (carried[at] & ~fmask) | s_kw[a] : s_kw[q * kCta + a];
                }
            }
            if (j == 0) continue;
            const uint32_t b = s_idx[j - 1];
            for (uint32_t q = 0; q < Wr; q++) {
                const uint32_t x = s_kw[q * kCta + a] ^ s_kw[q * kCta + b];
                if (x) {
                    const uint32_t d = moff[32u * (np - 1 - (uint32_t)(qtop - (int)q)) + (uint32_t)__clz(x)];
                    dbit[p0 + j] = (uint16_t)d;
                    const uint32_t bb = 0x80000000u >> (d & 31);
                    if (!(s_bm[d >> 5] & bb)) atomicOr(&s_bm[d >> 5], bb);
                    break;
                }
            }
        }
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x)
        if (s_bm[w]) atomicOr(&dacc[w], s_bm[w]);
}

// keep[k] = 1 for the members of unfinished runs except each run's first (the tie convention
// of the compaction), 0 otherwise
__global__ void __launch_bounds__(kRefThreads)
k_ref_keep(const uint32_t* __restrict__ seg, const uint32_t* __restrict__ run_off, const uint8_t* __restrict__ done,
           uint64_t nn, uint8_t* __restrict__ keep) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nn; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = seg[k];
        keep[k] = (!done[s] && run_off[s] != (uint32_t)k) ? 1 : 0;
    }
}

// A refinement round without LSD passes, when every long run fits a CTA: CTA per run (of the
// list made by the second compaction, runs in list order), its members' 64-bit chunk at bit o
// (from P_M by row id) and row ids staged in shared memory and bitonic-sorted by (chunk, row
// id) -- the stable order, as the (run, chunk) LSD round would produce -- then written in the
// LSD round's output format (compact planes lo, hi, run; sorted row ids) at the run's list range.
constexpr uint32_t kChunkCta = kChunkCtaKeys;
__global__ void __launch_bounds__(kRefThreads)
k_ref_cta_chunk(const uint32_t* __restrict__ pm, uint64_t pitch, uint32_t np, uint32_t o,
                const uint32_t* __restrict__ perm, const uint32_t* __restrict__ run_off,
                const uint32_t* __restrict__ run_pos, uint64_t nseg, uint64_t nn, uint32_t* __restrict__ out,
                uint64_t opitch, uint32_t* __restrict__ orid) {
    extern __shared__ uint32_t s_dyn[];
    uint32_t* s_hi = s_dyn;                                          // [kChunkCta]
    uint32_t* s_lo = s_hi + kChunkCta;
    uint32_t* s_row = s_lo + kChunkCta;
    uint16_t* s_idx = reinterpret_cast<uint16_t*>(s_row + kChunkCta);
    for (uint64_t s = blockIdx.x; s < nseg; s += gridDim.x) {
        const uint32_t k0 = run_off[s];
        const uint32_t k1 = s + 1 < nseg ? run_off[s + 1] : (uint32_t)nn;
        const uint32_t L = k1 - k0, p0 = run_pos[s];
        uint32_t P2 = 1;
        while (P2 < L) P2 <<= 1;
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < L; j += blockDim.x) {
            const uint32_t row = perm[p0 + j];
            s_row[j] = row;
            s_hi[j] = pm_bits32(pm, pitch, np, o, row);
            s_lo[j] = pm_bits32(pm, pitch, np, o + 32, row);
        }
        for (uint32_t j = threadIdx.x; j < P2; j += blockDim.x) s_idx[j] = (uint16_t)j;
        __syncthreads();
        auto less = [&](uint32_t a, uint32_t b) -> bool {            // padding (>= L) sorts last
            if (a >= L || b >= L) return a < b;
            if (s_hi[a] != s_hi[b]) return s_hi[a] < s_hi[b];
            if (s_lo[a] != s_lo[b]) return s_lo[a] < s_lo[b];
            return s_row[a] < s_row[b];
        };
        for (uint32_t size = 2; size <= P2; size <<= 1) {
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t i = threadIdx.x; i < P2 / 2; i += blockDim.x) {
                    const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    const uint32_t a = s_idx[lo], b = s_idx[hi];
                    if (less(b, a) == up) { s_idx[lo] = (uint16_t)b; s_idx[hi] = (uint16_t)a; }
                }
                __syncthreads();
            }
        }
        for (uint32_t j = threadIdx.x; j < L; j += blockDim.x) {
            const uint32_t a = s_idx[j];
            out[k0 + j] = s_lo[a];
            out[opitch + k0 + j] = s_hi[a];
            out[2 * opitch + k0 + j] = (uint32_t)s;
            orid[k0 + j] = s_row[a];
        }
    }
}

// sorted row ids back to their run's positions (and, when P_M is carried in sorted order,
// its planes for those rows)
__global__ void __launch_bounds__(kRefThreads)
k_ref_put(uint32_t* __restrict__ perm, const uint32_t* __restrict__ pos, const uint32_t* __restrict__ rid, uint64_t nr,
          const uint32_t* __restrict__ pm, uint64_t pitch, uint32_t np, uint32_t* __restrict__ carried) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nr; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = pos[k], r = rid[k];
        CKS_DCHECK(p < pitch && r < pitch);
        perm[p] = r;
        if (carried)
            for (uint32_t q = 0; q < np; q++) carried[(uint64_t)q * pitch + p] = __ldg(pm + (uint64_t)q * pitch + r);
    }
}

// the round-0 sorted planes (np0 of them, the top of P_M) at the listed positions, from P_M by
// the row id now there (the refinement reordered those positions; a7 repacks the planes)
__global__ void __launch_bounds__(kRefThreads)
k_ref_refresh(const uint32_t* __restrict__ list, uint64_t nr, const uint32_t* __restrict__ perm,
              const uint32_t* __restrict__ pm, uint64_t pitch, uint32_t np, uint32_t np0, uint32_t* __restrict__ sorted,
              uint64_t spitch) {
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nr; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t p = list[k], r = perm[p];
        CKS_DCHECK(p < spitch && r < pitch);
        for (uint32_t j = 0; j < np0; j++) sorted[(uint64_t)j * spitch + p] = __ldg(pm + (uint64_t)(np - np0 + j) * pitch + r);
    }
}

// ---- launchers --------------------------------------------------------------------------------

static unsigned grid_of(uint64_t work, int sms) {
    uint64_t g = (work + kRefThreads - 1) / kRefThreads;
    const uint64_t cap = (uint64_t)sms * 8;
    if (g > cap) g = cap;
    return (unsigned)(g ? g : 1);
}

// longest run sorted by one CTA (knob ref_cta, default 2048 = kCta)
static uint32_t cta_max() {
    const int v = knobs().ref_cta;
    return (uint32_t)(v < (int)kCta ? v : (int)kCta);
}

uint64_t ref_tiles(uint64_t nr) { return (nr + kRefTile - 1) / kRefTile; }

cudaError_t launch_ref_adj(const uint32_t* lo, const uint32_t* hi, const uint32_t* seg, const uint32_t* pos,
                           uint64_t nr, uint32_t cbase, const uint16_t* moff, uint32_t m, uint32_t B,
                           uint16_t* dbit, uint8_t* tie, uint32_t* dacc, bool round0, int sms, cudaStream_t st,
                           unsigned long long cmask) {
    if (nr == 0) return cudaSuccess;
    const uint32_t nwords = (8 * B + 31) / 32;
    const size_t smem = (size_t)nwords * 4 + (size_t)m * 2 + 16;
    k_ref_adj<<<grid_of(nr, sms), kRefThreads, smem, st>>>(lo, hi, seg, pos, nr, cbase, moff, m, nwords, dbit, tie,
                                                           dacc, round0 ? 1 : 0, cmask);
    return cudaGetLastError();
}

cudaError_t launch_ref_tile(const uint32_t* pm, uint64_t pitch, uint32_t np, int qtop, uint32_t fmask,
                            const uint16_t* moff, uint32_t* perm, uint16_t* dbit, uint32_t* carried, const uint32_t* lo,
                            const uint32_t* hi, uint64_t hpitch, uint64_t n, unsigned long long cmask, uint32_t B,
                            uint8_t* tie, uint32_t* dacc, uint32_t* handled, int sms, cudaStream_t st, uint8_t* any) {
    if (n == 0) return cudaSuccess;
    const uint32_t nwords = (8 * B + 31) / 32;
    RunCtx R{pm, pitch, np, qtop, fmask, moff, perm, dbit, carried};
    auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    const bool vec = al(perm) && al(dbit) && al(hi) && (!lo || al(lo)) && (hpitch & 3) == 0 && (pitch & 3) == 0 &&
                     (!carried || al(carried));
    if (!carried) return cudaErrorInvalidValue;
    const int wc = qtop + 1;
    const bool alias = (np == 3 || np == 4) && lo == carried + (np - 2) * pitch && hi == carried + (np - 1) * pitch;
    if (!alias) return cudaErrorInvalidValue;                    // (chunk = carried planes 2, 1)
    (void)nwords;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ref_reg<2, 3>, kRefThreads, 0);
    const uint64_t tiles = (n + kTileKeys - 1) / kTileKeys, gmax = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
    const unsigned rgrid = (unsigned)(tiles < gmax ? tiles : gmax);
#define CKS_TILE_CASE(W)                                                                                        \
    case W:                                                                                                     \
        if (np == 4) k_ref_reg<W < 3 ? W : 3, 4><<<rgrid, kRefThreads, 0, st>>>(R, lo, hi, n, cmask, vec, tie,   \
                                                                                dacc, handled, any);           \
        else k_ref_reg<W, 3><<<rgrid, kRefThreads, 0, st>>>(R, lo, hi, n, cmask, vec, tie, dacc, handled, any); \
        break;
    switch (wc) {
        CKS_TILE_CASE(1)
        CKS_TILE_CASE(2)
        CKS_TILE_CASE(3)
        default: return cudaErrorInvalidValue;
    }
#undef CKS_TILE_CASE
    return cudaGetLastError();
}

cudaError_t launch_ref_compact(const uint8_t* tie, uint64_t nr, const uint32_t* pos, uint32_t* cnt, uint32_t* tot,
                               uint32_t* pos_next, uint32_t* seg_next, uint32_t* run_off, uint32_t* run_pos,
                               cudaStream_t st, const uint8_t* any) {
    const uint64_t tiles = ref_tiles(nr);
    if (tiles == 0) return cudaMemsetAsync(tot, 0, 8, st);
    const unsigned grid = (unsigned)((tiles + kCompactTiles - 1) / kCompactTiles);
    k_ref_count<<<grid, kRefThreads, 0, st>>>(tie, nr, tiles, cnt, any);
    k_ref_scan<<<1, 1024, 0, st>>>(cnt, (uint32_t)tiles, tot);
    k_ref_scatter<1><<<(unsigned)tiles, kRefThreads, 0, st>>>(tie, nr, tiles, pos, cnt, pos_next, seg_next, run_off,
                                                             run_pos, any);
    return cudaGetLastError();
}

cudaError_t launch_ref_local(const uint32_t* pm, uint64_t pitch, uint32_t np, int qtop, const uint16_t* moff,
                             const uint32_t* run_pos, const uint32_t* seg, const uint32_t* run_off, uint64_t nseg,
                             uint64_t nn, uint32_t* perm, uint16_t* dbit, uint32_t* dacc, uint8_t* done, uint8_t* keep,
                             uint32_t* carried, uint32_t B, uint32_t* mlist, uint32_t* wlist, uint32_t* mcount, int sms,
                             cudaStream_t st, uint32_t fmask) {
    (void)seg;
    (void)keep;
    cudaMemsetAsync(mcount, 0, 16, st);                          // medium, long, warp runs; longest long run
    if (nseg == 0) return cudaGetLastError();
    const uint32_t nwords = (8 * B + 31) / 32;
    RunCtx R{pm, pitch, np, qtop, fmask, moff, perm, dbit, carried};
    k_ref_local<<<grid_of(nseg, sms), kRefThreads, 0, st>>>(R, run_pos, run_off, nseg, nn, dacc, done, nwords, mlist,
                                                            wlist, mcount, cta_max());
    if (qtop + 1 <= kRegWords)
        k_ref_warp<<<(unsigned)(sms * 8), kRefThreads, 0, st>>>(R, run_pos, run_off, nseg, nn, dacc, nwords, wlist, mcount);
    if (qtop + 1 <= (int)kCtaWords) {
        const size_t smem = (size_t)kCta * 4 * (qtop + 2) + (size_t)kCta * 2;
        raise_smem_limit((const void*)k_ref_cta, smem);
        k_ref_cta<<<(unsigned)(sms * 4), kRefThreads, smem, st>>>(pm, pitch, np, qtop, moff, run_pos, run_off, nseg, nn,
                                                                  perm, dbit, dacc, carried, nwords, mlist, mcount,
                                                                  fmask);
    }
    return cudaGetLastError();
}

cudaError_t launch_ref_keep(const uint32_t* seg, const uint32_t* run_off, const uint8_t* done, uint64_t nn,
                            uint8_t* keep, int sms, cudaStream_t st) {
    if (nn == 0) return cudaSuccess;
    k_ref_keep<<<grid_of(nn, sms), kRefThreads, 0, st>>>(seg, run_off, done, nn, keep);
    return cudaGetLastError();
}

cudaError_t launch_ref_gather(const uint32_t* pm, uint64_t pitch, uint32_t np, uint32_t o, const uint32_t* pos,
                              const uint32_t* seg, const uint32_t* perm, uint64_t nr, uint32_t* out, uint64_t opitch,
                              uint32_t* orid, int sms, cudaStream_t st) {
    if (nr == 0) return cudaSuccess;
    k_ref_gather<<<grid_of(nr, sms), kRefThreads, 0, st>>>(pm, pitch, np, o, pos, seg, perm, nr, out, opitch, orid);
    return cudaGetLastError();
}

cudaError_t launch_ref_cta_chunk(const uint32_t* pm, uint64_t pitch, uint32_t np, uint32_t o, const uint32_t* perm,
                                 const uint32_t* run_off, const uint32_t* run_pos, uint64_t nseg, uint64_t nn,
                                 uint32_t* out, uint64_t opitch, uint32_t* orid, int sms, cudaStream_t st) {
    if (nseg == 0) return cudaSuccess;
    const uint64_t g = nseg < (uint64_t)sms * 4 ? nseg : (uint64_t)sms * 4;
    const size_t smem = (size_t)kChunkCta * 14;
    raise_smem_limit((const void*)k_ref_cta_chunk, smem);
    k_ref_cta_chunk<<<(unsigned)g, kRefThreads, smem, st>>>(pm, pitch, np, o, perm, run_off, run_pos, nseg, nn, out,
                                                            opitch, orid);
    return cudaGetLastError();
}

cudaError_t launch_ref_refresh(const uint32_t* list, uint64_t nr, const uint32_t* perm, const uint32_t* pm,
                              uint64_t pitch, uint32_t np, uint32_t np0, uint32_t* sorted, uint64_t spitch, int sms,
                              cudaStream_t st) {
    if (nr == 0) return cudaSuccess;
    k_ref_refresh<<<grid_of(nr, sms), kRefThreads, 0, st>>>(list, nr, perm, pm, pitch, np, np0, sorted, spitch);
    return cudaGetLastError();
}

cudaError_t launch_ref_put(uint32_t* perm, const uint32_t* pos, const uint32_t* rid, uint64_t nr, const uint32_t* pm,
                           uint64_t pitch, uint32_t np, uint32_t* carried, int sms, cudaStream_t st) {
    if (nr == 0) return cudaSuccess;
    k_ref_put<<<grid_of(nr, sms), kRefThreads, 0, st>>>(perm, pos, rid, nr, pm, pitch, np, carried);
    return cudaGetLastError();
}

}  // namespace cks

namespace cks {

// One CTA: the top 64 bits of P_M of a strided sample of keys (compressed here with the
// compress plan, most significant gather step first) are bitonic-sorted in shared memory,
// then the number of distinct prefixes of the top 8, 16, ..., 64 bits is counted. Runs on a
// side stream while the full compress runs.
__global__ void __launch_bounds__(1024)
k_prefix_sample(const uint8_t* __restrict__ keys, uint64_t n, uint32_t B, const GatherPlan* __restrict__ plan,
                uint32_t S, uint32_t* __restrict__ counts, const uint32_t* __restrict__ pm, uint32_t np, uint64_t pitch) {
    extern __shared__ unsigned long long s_v[];                     // [S]
    __shared__ uint32_t s_cnt[8];
    if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
    const uint32_t nsteps = pm ? 0u : plan->nsteps;
    for (uint32_t i = threadIdx.x; i < S; i += blockDim.x) {
        if (pm) {                                                     // left-aligned P_M given
            const uint64_t r = (uint64_t)i * n / S;
            s_v[i] = ((unsigned long long)pm[(uint64_t)(np - 1) * pitch + r] << 32) |
                     (np >= 2 ? pm[(uint64_t)(np - 2) * pitch + r] : 0u);
            continue;
        }
        const uint8_t* k = keys + ((uint64_t)i * n / S) * B;
        unsigned long long top = 0;
        uint32_t got = 0;
        for (int s = (int)nsteps - 1; s >= 0 && got < 64; s--) {
            const GatherStep& g = plan->step[s];
            uint32_t w = 0;
            for (uint32_t b = 0; b < 4; b++) {
                const uint32_t j = g.src * 4 + b;
                w = (w << 8) | (j < B ? k[j] : 0u);
            }
            uint32_t x = w & g.mask;
#pragma unroll
            for (int q = 0; q < 5; q++) {
                const uint32_t tq = x & g.mv[q];
                x = (x ^ tq) | (tq >> (1u << q));
            }
            uint32_t c = g.cnt;
            if (got + c > 64) { x >>= got + c - 64; c = 64 - got; }
            top = (c == 64 ? 0ull : top << c) | x;
            got += c;
        }
        s_v[i] = got ? top << (64 - got) : 0ull;
    }
    __syncthreads();
    for (uint32_t size = 2; size <= S; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < S / 2; i += blockDim.x) {
                const uint32_t a = 2 * i - (i & (stride - 1)), b = a + stride;
                const bool up = (a & size) == 0;
                const unsigned long long x = s_v[a], y = s_v[b];
                if ((x > y) == up) { s_v[a] = y; s_v[b] = x; }
            }
            __syncthreads();
        }
    }
    uint32_t c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t i = threadIdx.x; i < S; i += blockDim.x) {
        const unsigned long long d = i ? s_v[i] ^ s_v[i - 1] : ~0ull;
#pragma unroll
        for (int w = 0; w < 8; w++) c[w] += (d >> (56 - 8 * w)) != 0;   // differs in the top 8(w+1) bits
    }
#pragma unroll
    for (int w = 0; w < 8; w++) {
        const uint32_t r = __reduce_add_sync(0xffffffffu, c[w]);
        if ((threadIdx.x & 31) == 0 && r) atomicAdd(&s_cnt[w], r);
    }
    __syncthreads();
    if (threadIdx.x < 8) counts[threadIdx.x] = s_cnt[threadIdx.x];
}

cudaError_t launch_prefix_sample(const uint8_t* keys, uint64_t n, uint32_t B, const GatherPlan* plan, uint32_t samples,
                                 uint32_t* counts, cudaStream_t st, const uint32_t* pm, uint32_t np, uint64_t pitch) {
    const size_t smem = (size_t)samples * 8;
    raise_smem_limit((const void*)k_prefix_sample, smem);
    k_prefix_sample<<<1, 1024, smem, st>>>(keys, n, B, plan, samples, counts, pm, np, pitch);
    return cudaGetLastError();
}

}  // namespace cks

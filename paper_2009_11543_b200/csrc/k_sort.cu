// k_sort.cu -- a4/a5: stable LSD radix sort of (P, row id) pairs.
//
// The paper sorts with its row-column comparison sort (App. A), a CPU design. Here the
// compressed keys are sorted by 8-bit digits, least significant first, one
// "onesweep"-style kernel per digit: each CTA takes a tile (dynamic tile id), ranks its
// keys by digit in shared memory, publishes its per-digit counts and resolves its global
// offsets by decoupled look-back over preceding tiles, then scatters keys and payload
// through shared memory so that runs of equal digits are written contiguously.
// Stability of every pass gives the row-id tie-break (reading R6).
//
// Layout: planes u32[np][n] (plane q = bits [32q, 32q+32) of P), payload u32 row id.
// Digit p of P = bits [8p, 8p+8) = byte (p & 3) of plane (p >> 2).
#include <stdlib.h>

#include "cks_internal.h"

namespace cks {

constexpr int kWarps = kSortThreads / 32;

// ------------------------------------------------------------------------------------
// digit histograms (all passes at once)

__global__ void __launch_bounds__(256)
k_hist(const uint32_t* __restrict__ planes, uint64_t pitch, uint64_t n, uint32_t key_passes,
       const uint32_t* __restrict__ rid, uint32_t rid_passes, uint32_t p0, uint32_t p1,
       uint32_t* __restrict__ hist) {
    extern __shared__ uint32_t h[];
    const uint32_t np_ = p1 - p0;
    for (uint32_t i = threadIdx.x; i < np_ * 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint32_t q0 = p0 >> 2;
    const uint32_t qk = (min(p1, key_passes) + 3) >> 2;   // key planes touched
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        for (uint32_t q = q0; q < qk; q++) {
            uint32_t w = planes[(uint64_t)q * pitch + i];
#pragma unroll
            for (uint32_t b = 0; b < 4; b++) {
                uint32_t p = q * 4 + b;
                if (p >= p0 && p < p1 && p < key_passes) atomicAdd(&h[(p - p0) * 256 + ((w >> (8 * b)) & 0xFF)], 1u);
            }
        }
        if (rid_passes && p1 > key_passes) {
            uint32_t w = rid[i];
            for (uint32_t b = 0; b < rid_passes; b++) {
                uint32_t p = key_passes + b;
                if (p >= p0 && p < p1) atomicAdd(&h[(p - p0) * 256 + ((w >> (8 * b)) & 0xFF)], 1u);
            }
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < np_ * 256; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[(uint64_t)p0 * 256 + i], h[i]);
}

cudaError_t launch_hist(const uint32_t* planes, uint64_t pitch, uint64_t n, uint32_t key_passes,
                        const uint32_t* rid, uint32_t rid_passes, uint32_t* hist, int sms,
                        cudaStream_t st, int* launches) {
    *launches = 0;
    const uint32_t total = key_passes + (rid ? rid_passes : 0);
    if (n == 0 || total == 0) return cudaSuccess;
    uint64_t want = (n + 255) / 256;
    const uint32_t group = 32;                              // passes per launch (32 KB smem)
    for (uint32_t p0 = 0; p0 < total; p0 += group) {
        uint32_t p1 = p0 + group < total ? p0 + group : total;
        int grid = (int)(want < (uint64_t)sms * 4 ? want : (uint64_t)sms * 4);
        k_hist<<<grid, 256, (size_t)(p1 - p0) * 256 * 4, st>>>(planes, pitch, n, key_passes, rid,
                                                              rid ? rid_passes : 0, p0, p1, hist);
        ++*launches;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// block-wide exclusive scan over 256 threads (one value each)

__device__ __forceinline__ uint32_t block_exclusive_scan256(uint32_t v, uint32_t* s_warp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t t = lane < kWarps ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < kWarps; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < kWarps) s_warp[lane] = t;               // inclusive warp totals
    }
    __syncthreads();
    uint32_t before = warp ? s_warp[warp - 1] : 0;
    return before + x - v;
}

__global__ void k_scan(const uint32_t* __restrict__ hist, uint32_t* __restrict__ base) {
    __shared__ uint32_t s_warp[kWarps];
    const uint32_t p = blockIdx.x;
    uint32_t v = hist[p * 256 + threadIdx.x];
    base[p * 256 + threadIdx.x] = block_exclusive_scan256(v, s_warp);
}

cudaError_t launch_scan(const uint32_t* hist, uint32_t passes, uint32_t* base, cudaStream_t st) {
    if (passes == 0) return cudaSuccess;
    k_scan<<<passes, 256, 0, st>>>(hist, base);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// one LSD pass

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// TMA (cp.async.bulk) helpers ------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    }
}

// Stream k of a pass: 0 = the word holding the digit, then the other planes in order,
// then the row id. Returns the plane index or -1 for the row id.
__device__ __forceinline__ int stream_id(int k, int dp, int np) {
    if (k == 0) return dp;
    int idx = k - 1;
    int others = np - (dp >= 0 ? 1 : 0);
    if (idx < others) return idx + ((dp >= 0 && idx >= dp) ? 1 : 0);
    return -1;
}

constexpr int kMaxSlots = 8;

// One stable LSD pass over one 8-bit digit ("onesweep"): CTA = one tile of kItems*256
// keys taken in dynamic order. All streams of the tile (digit word, other planes, row id)
// are fetched into shared-memory slots with 1-D TMA bulk copies issued by one thread, so
// the loads are in flight while the tile is ranked; slots are refilled as streams are
// consumed. The digit is ranked per warp (match_any; stable: item order, then lane order),
// counts are published and the tile's global offsets resolved by decoupled look-back over
// preceding tiles (status words: flag in the high half, count in the low half; flags
// carry the pass epoch so the array never needs clearing). Every stream is then permuted
// through shared memory into digit order and written out in coalesced runs.
template <int ITEMS, int RANK>
__global__ void __launch_bounds__(kSortThreads)
k_onesweep(const OnesweepArgs a) {
    constexpr int TILE = kSortThreads * ITEMS;
    extern __shared__ __align__(128) uint8_t s_dyn[];
    uint32_t* stage = reinterpret_cast<uint32_t*>(s_dyn);                 // [nslots][TILE]
    uint32_t* s_buf = stage + (size_t)a.slots * TILE;                        // [TILE]
    uint32_t (*s_hist)[kRadix] = reinterpret_cast<uint32_t (*)[kRadix]>(s_buf + TILE);  // [8][256]
    uint8_t* s_dig = reinterpret_cast<uint8_t*>(s_buf + TILE + kWarps * kRadix);        // [TILE]
    __shared__ uint32_t s_local[kRadix];
    __shared__ uint32_t s_gbase[kRadix];
    __shared__ uint32_t s_warp[kWarps];
    __shared__ uint32_t s_tile;
    __shared__ __align__(8) uint64_t s_bar[kMaxSlots];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t n = a.n;
    const int np = (int)a.nplanes, dp = a.digit_plane;
    const int S = np + 1;                                       // streams
    const int loaded = S - (a.in_rid == nullptr ? 1 : 0);       // implicit row id is last, never loaded
    const int nslots = loaded < (int)a.slots ? loaded : (int)a.slots;

    auto src_of = [&](int k) -> const uint32_t* {
        int id = stream_id(k, dp, np);
        return id >= 0 ? a.in_planes + (uint64_t)id * a.in_pitch : a.in_rid;
    };
    auto dst_of = [&](int k) -> uint32_t* {
        int id = stream_id(k, dp, np);
        return id >= 0 ? a.out_planes + (uint64_t)id * a.out_pitch : a.out_rid;
    };

    if (tid == 0) {
        uint32_t t = atomicAdd(a.tile_counter, 1u);
        s_tile = t;
        for (int sl = 0; sl < nslots; sl++) mbar_init(&s_bar[sl], 1);
        mbar_fence_init();
        const uint64_t b = (uint64_t)t * TILE;
        if (a.tma && b + TILE <= n)
            for (int k = 0; k < nslots; k++)
                tma_load_1d(stage + (size_t)k * TILE, src_of(k) + b, TILE * 4, &s_bar[k]);
    }
#pragma unroll
    for (int k = 0; k < kWarps; k++) s_hist[k][tid] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t base = (uint64_t)tile * TILE;
    const uint32_t tile_n = (uint32_t)(n - base < (uint64_t)TILE ? n - base : (uint64_t)TILE);
    const bool use_tma = a.tma && tile_n == (uint32_t)TILE;

    // streams are consumed in order 0, 1, 2, ...; stream k lives in slot k mod nslots and is
    // that slot's (k / nslots)-th fill, tracked incrementally (no division)
    int cur_slot = 0, cur_round = 0;
    auto acquire = [&](int k) -> const uint32_t* {
        uint32_t* slot = stage + (size_t)cur_slot * TILE;
        if (use_tma) {
            mbar_wait(&s_bar[cur_slot], (uint32_t)cur_round & 1u);
        } else {
            const uint32_t* src = src_of(k) + base;
            for (uint32_t i = tid; i < tile_n; i += kSortThreads) slot[i] = __ldg(src + i);
            __syncthreads();
        }
        return slot;
    };
    auto release = [&](int k_done) {                            // slot of k_done is free: refill it
        int nk = k_done + nslots;
        if (use_tma && tid == 0 && nk < loaded) {
            fence_proxy_async();
            tma_load_1d(stage + (size_t)cur_slot * TILE, src_of(nk) + base, TILE * 4, &s_bar[cur_slot]);
        }
        if (++cur_slot == nslots) { cur_slot = 0; cur_round++; }
    };

    // ---- rank the digit within each warp (warp-striped items: index w*32*ITEMS + i*32 + lane);
    // all match_any are issued back to back, then the per-warp counters are walked in item order
    const uint32_t* dslot = (dp < 0 && a.in_rid == nullptr) ? nullptr : acquire(0);
    const uint32_t wofs = (uint32_t)warp * 32 * ITEMS;
    uint32_t* h = s_hist[warp];
    const uint32_t ltm = lanemask_lt();
    uint32_t pos[ITEMS];
    uint32_t dg[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        uint32_t idx = wofs + i * 32 + lane;
        uint32_t key = idx < tile_n ? (dslot ? dslot[idx] : (uint32_t)(base + idx)) : 0u;
        dg[i] = idx < tile_n ? (key >> a.shift) & 0xFF : 0x100u;
    }
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        const bool valid = dg[i] < 0x100u;
        uint32_t peers;
        if (RANK == 0) {                       // intersect the 8 bit-plane ballots
            peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
            for (int b = 0; b < 8; b++) {
                uint32_t bit = (dg[i] >> b) & 1u;
                uint32_t bal = __ballot_sync(0xffffffffu, bit);
                peers &= bit ? bal : ~bal;
            }
        } else {
            peers = __match_any_sync(0xffffffffu, dg[i]);
            if (!valid) peers = 0;
        }
        // the group's leader (lowest lane) reserves popc(peers) slots of the warp's counter
        // for its digit; shared-memory atomics of one warp are applied in issue order, so
        // items keep their order without a per-item warp barrier
        const uint32_t lower = __popc(peers & ltm);
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (valid && lower == 0) old = atomicAdd(&h[dg[i]], (uint32_t)__popc(peers));
        old = __shfl_sync(0xffffffffu, old, leader < 0 ? lane : leader);
        pos[i] = old + lower;
    }
    __syncthreads();

    // ---- per digit (thread = digit): warp offsets and tile total; publish the aggregate
    uint32_t total = 0;
#pragma unroll
    for (int k = 0; k < kWarps; k++) {
        uint32_t c = s_hist[k][tid];
        s_hist[k][tid] = total;
        total += c;
    }
    const unsigned long long FA = (unsigned long long)(2u * a.epoch + 1u) << 32;
    const unsigned long long FP = (unsigned long long)(2u * a.epoch + 2u) << 32;
    unsigned long long* const col = a.status + tid;             // status of tile j, digit tid: col[j*256]
    st_relaxed_u64(col + (size_t)tile * kRadix, (tile == 0 ? FP : FA) | total);
    const uint32_t excl = block_exclusive_scan256(total, s_warp);
    s_local[tid] = excl;
    __syncthreads();

    // ---- stream 0 into tile (digit) order before the look-back: it needs local offsets only
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        if (dg[i] < 0x100u) {
            uint32_t idx = wofs + i * 32 + lane;
            uint32_t key = dslot ? dslot[idx] : (uint32_t)(base + idx);
            pos[i] += s_local[dg[i]] + s_hist[warp][dg[i]];
            s_buf[pos[i]] = key;
            s_dig[pos[i]] = (uint8_t)dg[i];
        }
    }

    // ---- decoupled look-back for digit tid, 8 predecessors per round trip
    {
        uint32_t prefix = 0;
        if (tile > 0 && !(a.debug & 1)) {
            int j = (int)tile - 1;                               // nearest predecessor not yet summed
            constexpr int WIN = 8;
            while (true) {
                unsigned long long v[WIN];
#pragma unroll
                for (int k = 0; k < WIN; k++)
                    v[k] = (j - k >= 0) ? ld_relaxed_u64(col + (uint32_t)(j - k) * kRadix) : FP;
                bool done = false;
                int k = 0;
                for (; k < WIN; k++) {
                    unsigned long long f = v[k] & 0xFFFFFFFF00000000ull;
                    if (f == FP) { prefix += (uint32_t)v[k]; done = true; break; }
                    if (f != FA) break;                          // not published yet: re-poll from here
                    prefix += (uint32_t)v[k];
                }
                if (done) break;
                if (k == 0) __nanosleep(16);                     // nearest one not ready: back off
                j -= k;
            }
            st_relaxed_u64(col + (size_t)tile * kRadix, FP | (unsigned long long)(prefix + total));
        }
        s_gbase[tid] = a.bucket_base[tid] + prefix - excl;
    }
    __syncthreads();
    if (dslot) release(0);
    uint32_t dest[ITEMS];
    {
        uint32_t* out = dst_of(0);
#pragma unroll
        for (int r = 0; r < ITEMS; r++) {
            uint32_t s = r * kSortThreads + tid;
            if (s < tile_n) {
                dest[r] = s_gbase[s_dig[s]] + s;
                out[dest[r]] = s_buf[s];
            }
        }
    }

    // ---- the other streams follow the same permutation
    for (int k = 1; k < ((a.debug & 2) ? 1 : S); k++) {
        __syncthreads();                                         // s_buf free again
        const bool implicit = k == S - 1 && a.in_rid == nullptr && dp >= 0;
        if (implicit) {
#pragma unroll
            for (int i = 0; i < ITEMS; i++)
                if (dg[i] < 0x100u) s_buf[pos[i]] = (uint32_t)(base + wofs + i * 32 + lane);
        } else {
            const uint32_t* slot = acquire(k);
#pragma unroll
            for (int i = 0; i < ITEMS; i++)
                if (dg[i] < 0x100u) s_buf[pos[i]] = slot[wofs + i * 32 + lane];
        }
        __syncthreads();
        if (!implicit) release(k);
        uint32_t* out = dst_of(k);
#pragma unroll
        for (int r = 0; r < ITEMS; r++) {
            uint32_t s = r * kSortThreads + tid;
            if (s < tile_n) out[dest[r]] = s_buf[s];
        }
    }
}

// Persistent variant: grid = resident CTAs; each CTA loops over dynamically claimed tiles.
// The shared-memory stream slots form one ring that runs across tile boundaries: when a
// stream is consumed its slot is refilled (TMA) with the next stream in sequence -- the
// next stream of this tile or the first streams of the tile claimed next -- so the loads
// of tile t+1 overlap the look-back and write-out of tile t. The next tile is claimed only
// once the current tile has published its aggregate (just before its look-back): claiming
// earlier makes later tiles wait on a claimed-but-unstarted tile. Each CTA processes its
// claims in order, so the smallest unfinished tile is always some CTA's current tile and
// the look-back cannot deadlock.
template <int ITEMS>
__global__ void __launch_bounds__(kSortThreads, ITEMS == 8 ? 4 : 2)
k_onesweep_persist(const OnesweepArgs a) {
    constexpr int TILE = kSortThreads * ITEMS;
    extern __shared__ __align__(128) uint8_t s_dyn[];
    uint32_t* ring = reinterpret_cast<uint32_t*>(s_dyn);                  // [R][TILE]
    uint32_t* s_buf = ring + (size_t)a.slots * TILE;                         // [TILE]
    uint32_t (*s_hist)[kRadix] = reinterpret_cast<uint32_t (*)[kRadix]>(s_buf + TILE);  // [8][256]
    uint8_t* s_dig = reinterpret_cast<uint8_t*>(s_buf + TILE + kWarps * kRadix);        // [TILE]
    __shared__ uint32_t s_local[kRadix];
    __shared__ uint32_t s_gbase[kRadix];
    __shared__ uint32_t s_warp[kWarps];
    __shared__ uint32_t s_cur;
    __shared__ __align__(8) uint64_t s_bar[kMaxSlots];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t n = a.n;
    const uint32_t ntiles = (uint32_t)((n + TILE - 1) / TILE);
    const int np = (int)a.nplanes, dp = a.digit_plane;
    const int S = np + 1;                                       // streams per tile
    const int L = S - (a.in_rid == nullptr ? 1 : 0);            // streams loaded per tile
    const int R = L < (int)a.slots ? L : (int)a.slots;          // ring slots (<= L: one tile ahead)

    auto src_of = [&](int k) -> const uint32_t* {
        int id = stream_id(k, dp, np);
        return id >= 0 ? a.in_planes + (uint64_t)id * a.in_pitch : a.in_rid;
    };
    auto dst_of = [&](int k) -> uint32_t* {
        int id = stream_id(k, dp, np);
        return id >= 0 ? a.out_planes + (uint64_t)id * a.out_pitch : a.out_rid;
    };
    auto full = [&](uint32_t t) { return a.tma && t < ntiles && (uint64_t)(t + 1) * TILE <= n; };

    // producer state (thread 0): next stream to issue is stream p_k of tile (p_sel ? next : cur)
    int p_k = 0, p_sel = 0, p_slot = 0;
    uint32_t t_cur = 0, t_next = 0;
    if (tid == 0) {
        for (int sl = 0; sl < R; sl++) mbar_init(&s_bar[sl], 1);
        mbar_fence_init();
        t_cur = atomicAdd(a.tile_counter, 1u);
        s_cur = t_cur;
        for (int sl = 0; sl < R; sl++) {                        // prologue: first R streams of t_cur
            if (full(t_cur)) tma_load_1d(ring + (size_t)sl * TILE, src_of(sl) + (uint64_t)t_cur * TILE, TILE * 4, &s_bar[sl]);
        }
        p_k = R;
        if (p_k == L) { p_k = 0; p_sel = 1; }
    }
    auto produce = [&]() {                                      // thread 0: refill slot p_slot
        const uint32_t t = p_sel ? t_next : t_cur;
        if (full(t)) {
            fence_proxy_async();
            tma_load_1d(ring + (size_t)p_slot * TILE, src_of(p_k) + (uint64_t)t * TILE, TILE * 4, &s_bar[p_slot]);
        }
        if (++p_slot == R) p_slot = 0;
        if (++p_k == L) { p_k = 0; p_sel++; }
    };

    int c_slot = 0, c_round = 0;                                // consumer ring position (all threads)
    const uint32_t wofs = (uint32_t)warp * 32 * ITEMS;
    const uint32_t ltm = lanemask_lt();
    const unsigned long long FA = (unsigned long long)(2u * a.epoch + 1u) << 32;
    const unsigned long long FP = (unsigned long long)(2u * a.epoch + 2u) << 32;
    unsigned long long* const col = a.status + tid;

    __syncthreads();
    while (true) {
        const uint32_t tile = s_cur;
        if (tile >= ntiles) break;
#pragma unroll
        for (int k = 0; k < kWarps; k++) s_hist[k][tid] = 0;
        const uint64_t base = (uint64_t)tile * TILE;
        const uint32_t tile_n = (uint32_t)(n - base < (uint64_t)TILE ? n - base : (uint64_t)TILE);
        const bool tma_t = full(tile);
        __syncthreads();

        auto acquire = [&](int k) -> const uint32_t* {
            uint32_t* slot = ring + (size_t)c_slot * TILE;
            if (tma_t) {
                mbar_wait(&s_bar[c_slot], (uint32_t)c_round & 1u);
            } else {
                const uint32_t* src = src_of(k) + base;
                for (uint32_t i = tid; i < tile_n; i += kSortThreads) slot[i] = __ldg(src + i);
                __syncthreads();
            }
            return slot;
        };
        auto release = [&]() {                                  // after a __syncthreads
            if (tid == 0) produce();
            if (++c_slot == R) { c_slot = 0; c_round++; }
        };

        // ---- rank (ballots; warp-striped items)
        const uint32_t* dslot = acquire(0);
        uint32_t* h = s_hist[warp];
        uint32_t pos[ITEMS];
        uint32_t dg[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; i++) {
            uint32_t idx = wofs + i * 32 + lane;
            dg[i] = idx < tile_n ? (dslot[idx] >> a.shift) & 0xFF : 0x100u;
        }
#pragma unroll
        for (int i = 0; i < ITEMS; i++) {
            const bool valid = dg[i] < 0x100u;
            uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
            for (int b = 0; b < 8; b++) {
                uint32_t bit = (dg[i] >> b) & 1u;
                uint32_t bal = __ballot_sync(0xffffffffu, bit);
                peers &= bit ? bal : ~bal;
            }
            uint32_t lower = __popc(peers & ltm);
            uint32_t cnt = valid ? h[dg[i]] : 0;
            pos[i] = cnt + lower;
            __syncwarp();
            if (valid && lower == 0) h[dg[i]] = cnt + __popc(peers);
            __syncwarp();
        }
        __syncthreads();

        // ---- per digit: warp offsets, tile total, publish aggregate, local scan
        uint32_t total = 0;
#pragma unroll
        for (int k = 0; k < kWarps; k++) {
            uint32_t c = s_hist[k][tid];
            s_hist[k][tid] = total;
            total += c;
        }
        st_relaxed_u64(col + (size_t)tile * kRadix, (tile == 0 ? FP : FA) | total);
        const uint32_t excl = block_exclusive_scan256(total, s_warp);
        s_local[tid] = excl;
        __syncthreads();

        // ---- stream 0 into digit order (local offsets only)
#pragma unroll
        for (int i = 0; i < ITEMS; i++) {
            if (dg[i] < 0x100u) {
                uint32_t idx = wofs + i * 32 + lane;
                pos[i] += s_local[dg[i]] + s_hist[warp][dg[i]];
                s_buf[pos[i]] = dslot[idx];
                s_dig[pos[i]] = (uint8_t)dg[i];
            }
        }

        if (tid == 0) t_next = atomicAdd(a.tile_counter, 1u);   // claim the next tile now
        // ---- decoupled look-back, 8 predecessors per round trip
        {
            uint32_t prefix = 0;
            if (tile > 0) {
                int j = (int)tile - 1;
                constexpr int WIN = 8;
                while (true) {
                    unsigned long long v[WIN];
#pragma unroll
                    for (int k = 0; k < WIN; k++)
                        v[k] = (j - k >= 0) ? ld_relaxed_u64(col + (uint32_t)(j - k) * kRadix) : FP;
                    bool done = false;
                    int k = 0;
                    for (; k < WIN; k++) {
                        unsigned long long f = v[k] & 0xFFFFFFFF00000000ull;
                        if (f == FP) { prefix += (uint32_t)v[k]; done = true; break; }
                        if (f != FA) break;
                        prefix += (uint32_t)v[k];
                    }
                    if (done) break;
                    if (k == 0) __nanosleep(16);
                    j -= k;
                }
                st_relaxed_u64(col + (size_t)tile * kRadix, FP | (unsigned long long)(prefix + total));
            }
            s_gbase[tid] = a.bucket_base[tid] + prefix - excl;
        }
        __syncthreads();
        release();
        uint32_t dest[ITEMS];
        {
            uint32_t* out = dst_of(0);
#pragma unroll
            for (int r = 0; r < ITEMS; r++) {
                uint32_t s = r * kSortThreads + tid;
                if (s < tile_n) {
                    dest[r] = s_gbase[s_dig[s]] + s;
                    out[dest[r]] = s_buf[s];
                }
            }
        }

        // ---- the other streams
        for (int k = 1; k < S; k++) {
            __syncthreads();
            const bool implicit = k == S - 1 && a.in_rid == nullptr;
            if (implicit) {
#pragma unroll
                for (int i = 0; i < ITEMS; i++)
                    if (dg[i] < 0x100u) s_buf[pos[i]] = (uint32_t)(base + wofs + i * 32 + lane);
            } else {
                const uint32_t* slot = acquire(k);
#pragma unroll
                for (int i = 0; i < ITEMS; i++)
                    if (dg[i] < 0x100u) s_buf[pos[i]] = slot[wofs + i * 32 + lane];
            }
            __syncthreads();
            if (!implicit) release();
            uint32_t* out = dst_of(k);
#pragma unroll
            for (int r = 0; r < ITEMS; r++) {
                uint32_t s = r * kSortThreads + tid;
                if (s < tile_n) out[dest[r]] = s_buf[s];
            }
        }
        __syncthreads();
        if (tid == 0) {                                          // advance: next becomes current
            t_cur = t_next;
            p_sel--;
            s_cur = t_cur;
        }
        __syncthreads();
    }
}

static int g_items = 0, g_slots = 0;                             // tuning overrides (env)

uint64_t onesweep_tile_keys() {
    if (!g_items) {
        const char* e = getenv("CKS_OS_ITEMS");
        g_items = e ? atoi(e) : 8;
        if (g_items != 8 && g_items != 16) g_items = 8;
        const char* s = getenv("CKS_OS_SLOTS");
        g_slots = s ? atoi(s) : 3;
        if (g_slots < 1) g_slots = 1;
        if (g_slots > kMaxSlots) g_slots = kMaxSlots;
    }
    return (uint64_t)kSortThreads * g_items;
}

uint64_t onesweep_tiles(uint64_t n) {
    uint64_t t = onesweep_tile_keys();
    return (n + t - 1) / t;
}

static int g_rank = -1;

template <int ITEMS, int RANK>
static cudaError_t launch_os(OnesweepArgs a, cudaStream_t st) {
    constexpr int TILE = kSortThreads * ITEMS;
    int streams = (int)a.nplanes + 1 - (a.in_rid == nullptr ? 1 : 0);
    if ((int)a.slots > streams) a.slots = streams > 0 ? streams : 1;
    size_t smem = (size_t)a.slots * TILE * 4 + (size_t)TILE * 4 + kWarps * kRadix * 4 + TILE;
    static size_t configured = 0;
    if (smem > configured) {
        cudaFuncSetAttribute(k_onesweep<ITEMS, RANK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    uint64_t tiles = (a.n + TILE - 1) / TILE;
    k_onesweep<ITEMS, RANK><<<(unsigned)tiles, kSortThreads, smem, st>>>(a);
    return cudaGetLastError();
}

static int g_persist = -1;

template <int ITEMS>
static cudaError_t launch_osp(OnesweepArgs a, cudaStream_t st) {
    constexpr int TILE = kSortThreads * ITEMS;
    int streams = (int)a.nplanes + 1 - (a.in_rid == nullptr ? 1 : 0);
    if ((int)a.slots > streams) a.slots = streams > 0 ? streams : 1;
    size_t smem = (size_t)a.slots * TILE * 4 + (size_t)TILE * 4 + kWarps * kRadix * 4 + TILE;
    static size_t configured = 0;
    static int dev_sms = 0;
    if (smem > configured) {
        cudaFuncSetAttribute(k_onesweep_persist<ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    if (!dev_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_onesweep_persist<ITEMS>, kSortThreads, smem);
    if (per_sm < 1) per_sm = 1;
    uint64_t tiles = (a.n + TILE - 1) / TILE;
    uint64_t grid = (uint64_t)dev_sms * per_sm;
    if (grid > tiles) grid = tiles;
    k_onesweep_persist<ITEMS><<<(unsigned)grid, kSortThreads, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_onesweep(const OnesweepArgs& args, cudaStream_t st) {
    if (args.n == 0) return cudaSuccess;
    OnesweepArgs a = args;
    onesweep_tile_keys();
    if (g_rank < 0) {
        const char* e = getenv("CKS_OS_RANK");
        g_rank = e ? (atoi(e) ? 1 : 0) : 0;
        const char* p = getenv("CKS_OS_PERSIST");
        g_persist = p ? (atoi(p) ? 1 : 0) : 1;
    }
    a.slots = (uint32_t)g_slots;
    static int dbg = -1;
    if (dbg < 0) { const char* e = getenv("CKS_OS_DEBUG"); dbg = e ? atoi(e) : 0; }
    a.debug = (uint32_t)dbg;
    // 1-D bulk copies need 16-byte aligned sources and plane strides
    a.tma = ((uintptr_t)a.in_planes % 16 == 0) && (a.in_pitch % 4 == 0) &&
            (a.in_rid == nullptr || (uintptr_t)a.in_rid % 16 == 0);
    if (g_persist) return g_items == 8 ? launch_osp<8>(a, st) : launch_osp<16>(a, st);
    if (g_items == 8) return g_rank ? launch_os<8, 1>(a, st) : launch_os<8, 0>(a, st);
    return g_rank ? launch_os<16, 1>(a, st) : launch_os<16, 0>(a, st);
}

}  // namespace cks

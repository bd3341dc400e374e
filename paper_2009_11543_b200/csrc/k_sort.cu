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
template <int ITEMS>
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
    const int nslots = loaded < a.slots ? loaded : a.slots;

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
    const uint64_t tile = s_tile;
    const uint64_t base = tile * TILE;
    const uint32_t tile_n = (uint32_t)(n - base < (uint64_t)TILE ? n - base : (uint64_t)TILE);
    const bool use_tma = a.tma && tile_n == (uint32_t)TILE;

    // make stream k available in its slot
    auto acquire = [&](int k) {
        uint32_t* slot = stage + (size_t)(k % nslots) * TILE;
        if (use_tma) {
            mbar_wait(&s_bar[k % nslots], (uint32_t)(k / nslots) & 1u);
        } else {
            const uint32_t* src = src_of(k) + base;
            for (uint32_t i = tid; i < tile_n; i += kSortThreads) slot[i] = __ldg(src + i);
            __syncthreads();
        }
        return slot;
    };
    auto refill = [&](int k_done) {                              // slot of k_done is free
        int nk = k_done + nslots;
        if (use_tma && tid == 0 && nk < loaded) {
            fence_proxy_async();
            tma_load_1d(stage + (size_t)(nk % nslots) * TILE, src_of(nk) + base, TILE * 4, &s_bar[nk % nslots]);
        }
    };

    // ---- rank the digit within each warp (warp-striped items: index w*32*ITEMS + i*32 + lane)
    const uint32_t* dslot = (dp < 0 && a.in_rid == nullptr) ? nullptr : acquire(0);
    const uint32_t wofs = (uint32_t)warp * 32 * ITEMS;
    uint32_t* h = s_hist[warp];
    const uint32_t ltm = lanemask_lt();
    uint32_t pos[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        uint32_t idx = wofs + i * 32 + lane;
        bool valid = idx < tile_n;
        uint32_t key = valid ? (dslot ? dslot[idx] : (uint32_t)(base + idx)) : 0u;
        uint32_t d = (key >> a.shift) & 0xFF;
        // peers = lanes with the same digit: intersect the 8 bit-plane ballots
        uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
        for (int b = 0; b < 8; b++) {
            uint32_t bit = (d >> b) & 1u;
            uint32_t bal = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? bal : ~bal;
        }
        uint32_t lower = __popc(peers & ltm);
        uint32_t cnt = valid ? h[d] : 0;
        pos[i] = cnt + lower;
        __syncwarp();
        if (valid && lower == 0) h[d] = cnt + __popc(peers);
        __syncwarp();
    }
    __syncthreads();

    // ---- per digit (thread = digit): warp offsets and tile total; publish the aggregate
    const uint32_t total = [&] {
        uint32_t t = 0;
#pragma unroll
        for (int k = 0; k < kWarps; k++) {
            uint32_t c = s_hist[k][tid];
            s_hist[k][tid] = t;
            t += c;
        }
        return t;
    }();
    const unsigned long long FA = (unsigned long long)(2u * a.epoch + 1u) << 32;
    const unsigned long long FP = (unsigned long long)(2u * a.epoch + 2u) << 32;
    unsigned long long* my = a.status + tile * kRadix + tid;
    st_relaxed_u64(my, (tile == 0 ? FP : FA) | total);
    const uint32_t excl = block_exclusive_scan256(total, s_warp);
    s_local[tid] = excl;
    __syncthreads();

    // ---- stream 0 into tile (digit) order before the look-back: it needs local offsets only
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        uint32_t idx = wofs + i * 32 + lane;
        if (idx < tile_n) {
            uint32_t key = dslot ? dslot[idx] : (uint32_t)(base + idx);
            uint32_t d = (key >> a.shift) & 0xFF;
            pos[i] += s_local[d] + s_hist[warp][d];
            s_buf[pos[i]] = key;
            s_dig[pos[i]] = (uint8_t)d;
        }
    }

    // ---- decoupled look-back for digit tid, 8 predecessors per round trip
    {
        uint32_t prefix = 0;
        if (tile > 0) {
            int64_t j = (int64_t)tile - 1;                       // nearest predecessor not yet summed
            constexpr int WIN = 8;
            while (true) {
                unsigned long long v[WIN];
#pragma unroll
                for (int k = 0; k < WIN; k++)
                    v[k] = (j - k >= 0) ? ld_relaxed_u64(a.status + (uint64_t)(j - k) * kRadix + tid) : FP;
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
            st_relaxed_u64(my, FP | (unsigned long long)(prefix + total));
        }
        s_gbase[tid] = a.bucket_base[tid] + prefix - excl;
    }
    __syncthreads();
    if (dslot) refill(0);
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
    for (int k = 1; k < S; k++) {
        __syncthreads();                                         // s_buf free again
        const bool implicit = stream_id(k, dp, np) < 0 && a.in_rid == nullptr;
        if (implicit) {
#pragma unroll
            for (int i = 0; i < ITEMS; i++) {
                uint32_t idx = wofs + i * 32 + lane;
                if (idx < tile_n) s_buf[pos[i]] = (uint32_t)(base + idx);
            }
        } else {
            const uint32_t* slot = acquire(k);
#pragma unroll
            for (int i = 0; i < ITEMS; i++) {
                uint32_t idx = wofs + i * 32 + lane;
                if (idx < tile_n) s_buf[pos[i]] = slot[idx];
            }
        }
        __syncthreads();
        if (!implicit) refill(k);
        uint32_t* out = dst_of(k);
#pragma unroll
        for (int r = 0; r < ITEMS; r++) {
            uint32_t s = r * kSortThreads + tid;
            if (s < tile_n) out[dest[r]] = s_buf[s];
        }
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

template <int ITEMS>
static cudaError_t launch_os(OnesweepArgs a, cudaStream_t st) {
    constexpr int TILE = kSortThreads * ITEMS;
    int streams = (int)a.nplanes + 1 - (a.in_rid == nullptr ? 1 : 0);
    if (a.slots > streams) a.slots = streams > 0 ? streams : 1;
    size_t smem = (size_t)a.slots * TILE * 4 + (size_t)TILE * 4 + kWarps * kRadix * 4 + TILE;
    static size_t configured = 0;
    if (smem > configured) {
        cudaFuncSetAttribute(k_onesweep<ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    uint64_t tiles = (a.n + TILE - 1) / TILE;
    k_onesweep<ITEMS><<<(unsigned)tiles, kSortThreads, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_onesweep(const OnesweepArgs& args, cudaStream_t st) {
    if (args.n == 0) return cudaSuccess;
    OnesweepArgs a = args;
    onesweep_tile_keys();
    a.slots = (uint32_t)g_slots;
    // 1-D bulk copies need 16-byte aligned sources and plane strides
    a.tma = ((uintptr_t)a.in_planes % 16 == 0) && (a.in_pitch % 4 == 0) &&
            (a.in_rid == nullptr || (uintptr_t)a.in_rid % 16 == 0);
    if (g_items == 8) return launch_os<8>(a, st);
    return launch_os<16>(a, st);
}

}  // namespace cks

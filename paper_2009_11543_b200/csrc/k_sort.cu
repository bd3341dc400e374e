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
#include "cks_internal.h"

namespace cks {

constexpr int kItems = 16;                               // keys per thread per tile
constexpr int kTile = kSortThreads * kItems;             // 4096 keys
constexpr int kWarps = kSortThreads / 32;

uint64_t onesweep_tiles(uint64_t n) { return (n + kTile - 1) / kTile; }

// ------------------------------------------------------------------------------------
// digit histograms (all passes at once)

__global__ void __launch_bounds__(256)
k_hist(const uint32_t* __restrict__ planes, uint64_t n, uint32_t key_passes,
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
            uint32_t w = planes[(uint64_t)q * n + i];
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

cudaError_t launch_hist(const uint32_t* planes, uint64_t n, uint32_t key_passes,
                        const uint32_t* rid, uint32_t rid_passes, uint32_t* hist, int sms,
                        cudaStream_t st) {
    const uint32_t total = key_passes + (rid ? rid_passes : 0);
    if (n == 0 || total == 0) return cudaSuccess;
    uint64_t want = (n + 255) / 256;
    const uint32_t group = 32;                              // passes per launch (32 KB smem)
    for (uint32_t p0 = 0; p0 < total; p0 += group) {
        uint32_t p1 = p0 + group < total ? p0 + group : total;
        int grid = (int)(want < (uint64_t)sms * 4 ? want : (uint64_t)sms * 4);
        k_hist<<<grid, 256, (size_t)(p1 - p0) * 256 * 4, st>>>(planes, n, key_passes, rid,
                                                              rid ? rid_passes : 0, p0, p1, hist);
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

__global__ void __launch_bounds__(kSortThreads)
k_onesweep(const OnesweepArgs a) {
    __shared__ uint32_t s_hist[kWarps][kRadix];      // per-warp digit counts -> warp offsets
    __shared__ uint32_t s_local[kRadix];             // tile-local exclusive digit offsets
    __shared__ uint32_t s_gbase[kRadix];             // global position of smem slot 0 per digit
    __shared__ uint32_t s_warp[kWarps];
    __shared__ uint32_t s_buf[kTile];                // exchange buffer
    __shared__ uint32_t s_tile;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t n = a.n;
    if (tid == 0) s_tile = atomicAdd(a.tile_counter, 1u);
#pragma unroll
    for (int k = 0; k < kWarps; k++) s_hist[k][tid] = 0;
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t base = tile * kTile;
    const uint32_t tile_n = (uint32_t)(n - base < (uint64_t)kTile ? n - base : (uint64_t)kTile);
    const uint64_t wbase = base + (uint64_t)warp * 32 * kItems;

    // ---- load the digit word of each key (warp-striped: coalesced 128-byte rows)
    const uint32_t* dsrc = a.digit_plane >= 0 ? a.in_planes + (uint64_t)a.digit_plane * n : a.in_rid;
    uint32_t key[kItems];
    uint32_t pos[kItems];
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        uint64_t idx = wbase + i * 32 + lane;
        key[i] = idx < n ? (dsrc ? __ldg(dsrc + idx) : (uint32_t)idx) : 0u;
    }

    // ---- rank within the warp (stable: item order, then lane order)
    uint32_t* h = s_hist[warp];
    const uint32_t ltm = lanemask_lt();
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        uint64_t idx = wbase + i * 32 + lane;
        bool valid = idx < n;
        uint32_t d = valid ? (key[i] >> a.shift) & 0xFF : 0x100u;
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t lower = __popc(peers & ltm);
        uint32_t cnt = valid ? h[d] : 0;
        pos[i] = cnt + lower;
        __syncwarp();
        if (valid && lower == 0) h[d] = cnt + __popc(peers);
        __syncwarp();
    }
    __syncthreads();

    // ---- per digit (thread = digit): warp offsets, tile total, publish, look-back
    const uint32_t d = tid;
    uint32_t total = 0;
#pragma unroll
    for (int k = 0; k < kWarps; k++) {
        uint32_t c = s_hist[k][d];
        s_hist[k][d] = total;
        total += c;
    }
    const unsigned long long FA = (unsigned long long)(2u * a.epoch + 1u) << 32;
    const unsigned long long FP = (unsigned long long)(2u * a.epoch + 2u) << 32;
    unsigned long long* my = a.status + tile * kRadix + d;
    if (tile == 0) st_relaxed_u64(my, FP | total);
    else st_relaxed_u64(my, FA | total);
    uint32_t excl = block_exclusive_scan256(total, s_warp);
    s_local[d] = excl;
    uint32_t prefix = 0;
    if (tile > 0) {
        int64_t j = (int64_t)tile - 1;
        while (true) {
            unsigned long long v = ld_relaxed_u64(a.status + (uint64_t)j * kRadix + d);
            unsigned long long f = v & 0xFFFFFFFF00000000ull;
            if (f == FP) { prefix += (uint32_t)v; break; }
            if (f == FA) { prefix += (uint32_t)v; j--; continue; }
            __nanosleep(32);
        }
        st_relaxed_u64(my, FP | (unsigned long long)(prefix + total));
    }
    s_gbase[d] = a.bucket_base[d] + prefix - excl;
    __syncthreads();

    // ---- scatter the digit word into tile order
#pragma unroll
    for (int i = 0; i < kItems; i++) {
        uint64_t idx = wbase + i * 32 + lane;
        if (idx < n) {
            uint32_t dd = (key[i] >> a.shift) & 0xFF;
            pos[i] += s_local[dd] + s_hist[warp][dd];
            s_buf[pos[i]] = key[i];
        }
    }
    __syncthreads();
    uint32_t dest[kItems];
    uint32_t* dout = a.digit_plane >= 0 ? a.out_planes + (uint64_t)a.digit_plane * n : a.out_rid;
#pragma unroll
    for (int r = 0; r < kItems; r++) {
        uint32_t s = r * kSortThreads + tid;
        if (s < tile_n) {
            uint32_t v = s_buf[s];
            dest[r] = s_gbase[(v >> a.shift) & 0xFF] + s;
            dout[dest[r]] = v;
        }
    }

    // ---- the other planes and the row id follow the same permutation
    const int nstreams = (int)a.nplanes + 1;             // planes 0..np-1, then row id
    for (int q = 0; q < nstreams; q++) {
        const bool is_rid = q == (int)a.nplanes;
        if (is_rid ? a.digit_plane < 0 : q == a.digit_plane) continue;
        const uint32_t* src = is_rid ? a.in_rid : a.in_planes + (uint64_t)q * n;
        uint32_t* dst = is_rid ? a.out_rid : a.out_planes + (uint64_t)q * n;
        uint32_t v[kItems];
#pragma unroll
        for (int i = 0; i < kItems; i++) {
            uint64_t idx = wbase + i * 32 + lane;
            v[i] = idx < n ? (src ? __ldg(src + idx) : (uint32_t)idx) : 0u;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kItems; i++) {
            uint64_t idx = wbase + i * 32 + lane;
            if (idx < n) s_buf[pos[i]] = v[i];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kItems; r++) {
            uint32_t s = r * kSortThreads + tid;
            if (s < tile_n) dst[dest[r]] = s_buf[s];
        }
    }
}

cudaError_t launch_onesweep(const OnesweepArgs& a, cudaStream_t st) {
    if (a.n == 0) return cudaSuccess;
    uint64_t tiles = onesweep_tiles(a.n);
    k_onesweep<<<(unsigned)tiles, kSortThreads, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace cks

// k_compress.cu -- a3: Compress(key) = the key's bits at the mask positions,
// concatenated in position order (extraction pipeline Sec. 5.1),
// and a7: repack of sorted P_M to P_D.
//
// The paper extracts with x86 PEXT on 8-byte mask segments. There is no
// PEXT on the GPU; each 32-bit big-endian key word with a non-zero mask word is
// compressed in registers with five masked shifts (parallel-suffix compress; move
// masks precomputed on the host per word), and the fields are appended from the least
// significant end of P upward, emitting a u32 plane whenever 32 bits are complete.
//
// Layout: keys u8[n][B] -> planes u32[np][n] (plane q = bits [32q, 32q+32) of P).
// Keys are staged through shared memory with coalesced 16-byte loads; each row is
// padded to an odd number of 16-byte units so a thread's 16-byte reads of its own row
// are bank-conflict free (8 lanes per phase hit 8 distinct 16-byte bank groups).
#include <stdlib.h>
#include <string.h>

#include <utility>

#include "cks_internal.h"
#include "k_occ_flags.cuh"

namespace cks {

__device__ __forceinline__ int4 ld_stream16c(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

__device__ __forceinline__ uint32_t gather_word(uint32_t x, const GatherStep& s) {
    x &= s.mask;
#pragma unroll
    for (int k = 0; k < 5; k++) {
        uint32_t t = x & s.mv[k];
        x = (x ^ t) | (t >> (1u << k));
    }
    return x;
}

constexpr int kCompressThreads = 256;

// B % 16 == 0 and keys 16-byte aligned: shared-memory staged tile of 256 keys.
__global__ void __launch_bounds__(kCompressThreads)
k_compress_tiled(const uint8_t* __restrict__ keys, uint64_t n, uint32_t B,
                 const GatherPlan* __restrict__ plan, uint32_t nsteps, uint32_t np,
                 uint32_t* __restrict__ planes, uint64_t pitch, uint32_t lead) {
    extern __shared__ int4 s_tile[];                      // [256][S16] int4 units
    __shared__ GatherStep s_step[kMaxWords];
    for (uint32_t s = threadIdx.x; s < nsteps; s += blockDim.x) s_step[s] = plan->step[s];
    const uint32_t U = B >> 4;                            // 16-byte units per key
    const uint32_t S16 = U | 1;                           // odd row stride (units)
    const uint64_t ntiles = (n + kCompressThreads - 1) / kCompressThreads;
    __syncthreads();
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t k0 = tile * kCompressThreads;
        const uint32_t tk = (uint32_t)(n - k0 < (uint64_t)kCompressThreads ? n - k0 : (uint64_t)kCompressThreads);
        const int4* src = reinterpret_cast<const int4*>(keys + k0 * B);
        const uint32_t units = tk * U;
        for (uint32_t c = threadIdx.x; c < units; c += kCompressThreads) {
            uint32_t r = c / U, u = c - r * U;
            s_tile[r * S16 + u] = ld_stream16c(src + c);
        }
        __syncthreads();
        if (threadIdx.x < tk) {
            const int4* row = s_tile + threadIdx.x * S16;
            const uint64_t i = k0 + threadIdx.x;
            unsigned long long acc = 0;
            uint32_t accbits = lead, q = 0;
            int cur_u = -1;
            int4 cur = make_int4(0, 0, 0, 0);
            for (uint32_t s = 0; s < nsteps; s++) {
                const GatherStep& g = s_step[s];
                int u = (int)(g.src >> 2);
                if (u != cur_u) { cur = row[u]; cur_u = u; }
                uint32_t sel = g.src & 3;
                uint32_t w = sel == 0 ? (uint32_t)cur.x : sel == 1 ? (uint32_t)cur.y
                           : sel == 2 ? (uint32_t)cur.z : (uint32_t)cur.w;
                uint32_t x = gather_word(bswap32(w), g);
                acc |= (unsigned long long)x << accbits;
                accbits += g.cnt;
                if (accbits >= 32) {
                    planes[(uint64_t)q * pitch + i] = (uint32_t)acc;
                    acc >>= 32;
                    accbits -= 32;
                    q++;
                }
            }
            if (accbits) planes[(uint64_t)q * pitch + i] = (uint32_t)acc;
        }
        __syncthreads();
    }
}

// Generic path: any B (word assembled from bytes, zero beyond B), any alignment.
__global__ void __launch_bounds__(kCompressThreads)
k_compress_generic(const uint8_t* __restrict__ keys, uint64_t n, uint32_t B,
                   const GatherPlan* __restrict__ plan, uint32_t nsteps, uint32_t np,
                   uint32_t* __restrict__ planes, uint64_t pitch, uint32_t lead, const uint32_t* __restrict__ rows) {
    __shared__ GatherStep s_step[kMaxWords];
    for (uint32_t s = threadIdx.x; s < nsteps; s += blockDim.x) s_step[s] = plan->step[s];
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint8_t* k = keys + (rows ? (uint64_t)rows[i] : i) * B;
        unsigned long long acc = 0;
        uint32_t accbits = lead, q = 0;
        for (uint32_t s = 0; s < nsteps; s++) {
            const GatherStep& g = s_step[s];
            uint32_t w = 0;
            for (uint32_t b = 0; b < 4; b++) {
                uint32_t j = g.src * 4 + b;
                w = (w << 8) | (j < B ? k[j] : 0u);
            }
            uint32_t x = gather_word(w, g);
            acc |= (unsigned long long)x << accbits;
            accbits += g.cnt;
            if (accbits >= 32) {
                planes[(uint64_t)q * pitch + i] = (uint32_t)acc;
                acc >>= 32;
                accbits -= 32;
                q++;
            }
        }
        if (accbits) planes[(uint64_t)q * pitch + i] = (uint32_t)acc;
    }
}

// a7 repack: source words are the planes of P_M (plane 0 least significant), each
// gathered by the sub-mask of P_M bits that are exact-D positions.
__global__ void __launch_bounds__(kCompressThreads)
k_repack(const uint32_t* __restrict__ in, uint64_t in_pitch, uint64_t n, const GatherPlan* __restrict__ plan,
         uint32_t nsteps, uint32_t np, uint32_t* __restrict__ out, uint64_t out_pitch, const uint32_t* __restrict__ rows) {
    __shared__ GatherStep s_step[kMaxPlanes];
    for (uint32_t s = threadIdx.x; s < nsteps; s += blockDim.x) s_step[s] = plan->step[s];
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        unsigned long long acc = 0;
        uint32_t accbits = 0, q = 0;
        for (uint32_t s = 0; s < nsteps; s++) {
            const GatherStep& g = s_step[s];
            uint32_t x = gather_word(in[(uint64_t)g.src * in_pitch + (rows ? (uint64_t)rows[i] : i)], g);
            acc |= (unsigned long long)x << accbits;
            accbits += g.cnt;
            if (accbits >= 32) {
                out[(uint64_t)q * out_pitch + i] = (uint32_t)acc;
                acc >>= 32;
                accbits -= 32;
                q++;
            }
        }
        if (accbits) out[(uint64_t)q * out_pitch + i] = (uint32_t)acc;
    }
}

// Fixed key width B in {8, 16, 32, 64}, 16-byte aligned keys: the per-word gather masks are
// a kernel parameter (constant bank) indexed by compile-time word numbers, the word loop is
// fully unrolled, and each thread loads its own key with 8- or 16-byte loads (for B >= 32 the
// later loads of a key hit the sectors its first load brought into L1).
template <int NW>
struct FixedPlan {
    uint32_t mask[NW];
    uint32_t mv[NW][5];
    uint32_t cnt[NW];
};

template <int B>
__device__ __forceinline__ void load_key(const uint8_t* kp, uint32_t (&w)[B / 4]) {
    if (B == 8) {
        uint2 v = __ldg(reinterpret_cast<const uint2*>(kp));
        w[0] = v.x;
        w[1] = v.y;
    } else {
#pragma unroll
        for (int u = 0; u < B / 16; u++) {
            uint4 v = __ldg(reinterpret_cast<const uint4*>(kp) + u);
            w[4 * u + 0] = v.x;
            w[4 * u + 1] = v.y;
            w[4 * u + 2] = v.z;
            w[4 * u + 3] = v.w;
        }
    }
}

__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// KPT keys per thread per iteration, all loads issued before any gather: more bytes in
// flight (the row-list variant's loads are random rows behind a dependent perm load).
// The gather runs mirrored (move_masks_left): each field ends left-aligned in its word and
// a step is one multiply-add, x + (x & mv) * (2^(2^s) - 1) (the moved bits land on zeros,
// so the add is the OR of the shifted bits), which runs on the FMA pipe and halves the
// integer-ALU work that bounds this kernel; the fields are appended from the most
// significant end of P down, plane np-1 first, after `toppad` zero bits.
template <int B, int KPT>
__global__ void __launch_bounds__(kCompressThreads)
k_compress_fixed(const uint8_t* __restrict__ keys, uint64_t n, const __grid_constant__ FixedPlan<B / 4> plan,
                 uint32_t* __restrict__ planes, uint64_t pitch, uint32_t np, uint32_t toppad,
                 const uint32_t* __restrict__ rows) {
    constexpr int NW = B / 4;
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += T * KPT) {
        uint32_t w[KPT][NW];
        uint64_t r[KPT];
#pragma unroll
        for (int u = 0; u < KPT; u++) {
            const uint64_t i = i0 + u * T;
            r[u] = i < n ? (rows ? (uint64_t)__ldg(rows + i) : i) : 0;
        }
#pragma unroll
        for (int u = 0; u < KPT; u++)
            if (i0 + u * T < n) load_key<B>(keys + r[u] * B, w[u]);
#pragma unroll
        for (int u = 0; u < KPT; u++) {
            const uint64_t i = i0 + u * T;
            if (i >= n) break;
            unsigned long long acc = 0;                          // pending bits, left-aligned
            uint32_t accbits = toppad, q = np - 1;
#pragma unroll
            for (int k = 0; k < NW; k++) {                       // most significant end of P first
                if (plan.mask[k] == 0) continue;
                uint32_t x = bswap32(w[u][k]) & plan.mask[k];
#pragma unroll
                for (int s = 0; s < 5; s++) x = mad_u32(x & plan.mv[k][s], (1u << (1u << s)) - 1u, x);
                acc |= ((unsigned long long)x << 32) >> accbits;
                accbits += plan.cnt[k];
                if (accbits >= 32) {
                    planes[(uint64_t)q * pitch + i] = (uint32_t)(acc >> 32);
                    acc <<= 32;
                    accbits -= 32;
                    q--;
                }
            }
            if (accbits) planes[(uint64_t)q * pitch + i] = (uint32_t)(acc >> 32);
        }
    }
}

// The speculative first build's compress (cks_api.cu build_common): k_compress_fixed<B, 1>
// by a mask taken from a sample of the rows, marking every key byte's occupancy on the way (the
// byte-occupancy superset pass fused into the compress: the keys are read once). The caller
// compares the full occupancy's D+ with the mask afterwards and compresses again if they differ.
template <int B>
__global__ void __launch_bounds__(kCompressThreads)
k_compress_occ(const uint8_t* __restrict__ keys, uint64_t n, const __grid_constant__ FixedPlan<B / 4> plan,
               uint32_t* __restrict__ planes, uint64_t pitch, uint32_t np, uint32_t toppad, uint32_t* __restrict__ occ) {
    constexpr int NW = B / 4;
    __shared__ __align__(16) uint8_t flag[B * kRowBytes];
    for (uint32_t i = threadIdx.x; i < B * kRowBytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(flag)[i] = 0;
    __syncthreads();
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += T) {
        uint32_t w[NW];
        load_key<B>(keys + i * B, w);
#pragma unroll
        for (int k = 0; k < NW; k++)
#pragma unroll
            for (int b = 0; b < 4; b++) flag[(4 * k + b) * kRowBytes + __byte_perm(w[k], 0, 0x4440 + b)] = 1;
        unsigned long long acc = 0;                          // pending bits, left-aligned
        uint32_t accbits = toppad, q = np - 1;
#pragma unroll
        for (int k = 0; k < NW; k++) {                       // most significant end of P first
            if (plan.mask[k] == 0) continue;
            uint32_t x = bswap32(w[k]) & plan.mask[k];
#pragma unroll
            for (int s = 0; s < 5; s++) x = mad_u32(x & plan.mv[k][s], (1u << (1u << s)) - 1u, x);
            acc |= ((unsigned long long)x << 32) >> accbits;
            accbits += plan.cnt[k];
            if (accbits >= 32) {
                planes[(uint64_t)q * pitch + i] = (uint32_t)(acc >> 32);
                acc <<= 32;
                accbits -= 32;
                q--;
            }
        }
        if (accbits) planes[(uint64_t)q * pitch + i] = (uint32_t)(acc >> 32);
    }
    __syncthreads();
    fold_flags<B>(flag, occ);
}

// Uniform-width masks (every key word holds C mask bits, e.g. cfg5's ACGT: 3 bits a byte, 12 a
// word; cfg3: 28) with P_M left-aligned (no top padding): every field's plane and shift are
// compile-time, so the plane words are assembled by constant shifts and stored once each -- no
// running bit count, no per-word plane test (k_compress_fixed / k_compress_occ keep those for
// any mask). OCC: also marks the byte occupancy as k_compress_occ does.
template <int B, int C, bool OCC>
__global__ void __launch_bounds__(kCompressThreads)
k_compress_uni(const uint8_t* __restrict__ keys, uint64_t n, const __grid_constant__ FixedPlan<B / 4> plan,
               uint32_t* __restrict__ planes, uint64_t pitch, uint32_t* __restrict__ occ) {
    constexpr int NW = B / 4, M = NW * C, NP = (M + 31) / 32;
    __shared__ __align__(16) uint8_t flag[OCC ? B * kRowBytes : 16];
    if (OCC) {
        for (uint32_t i = threadIdx.x; i < B * kRowBytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(flag)[i] = 0;
        __syncthreads();
    }
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += T) {
        uint32_t w[NW];
        load_key<B>(keys + i * B, w);
        if (OCC) {
#pragma unroll
            for (int k = 0; k < NW; k++)
#pragma unroll
                for (int b = 0; b < 4; b++) flag[(4 * k + b) * kRowBytes + __byte_perm(w[k], 0, 0x4440 + b)] = 1;
        }
        uint32_t out[NP];
#pragma unroll
        for (int q = 0; q < NP; q++) out[q] = 0;
#pragma unroll
        for (int k = 0; k < NW; k++) {
            uint32_t x = bswap32(w[k]) & plan.mask[k];
#pragma unroll
            for (int s = 0; s < 5; s++) x = mad_u32(x & plan.mv[k][s], (1u << (1u << s)) - 1u, x);
            // x: the word's C-bit field, left-aligned; it starts at bit k*C of P_M (from the MSB)
            const int off = k * C, q = NP - 1 - off / 32, r = off % 32;
            out[q] |= r ? x >> r : x;
            if (r + C > 32) out[q - 1] |= x << (32 - r);
        }
#pragma unroll
        for (int q = 0; q < NP; q++) planes[(uint64_t)q * pitch + i] = out[q];
    }
    if (OCC) {
        __syncthreads();
        fold_flags<B>(flag, occ);
    }
}

template <int B, int C>
static void launch_uni_c(const uint8_t* keys, uint64_t n, const FixedPlan<B / 4>& fp, uint32_t* planes, uint64_t pitch,
                         int grid, cudaStream_t st, uint32_t* occ) {
    if (occ) k_compress_uni<B, C, true><<<grid, kCompressThreads, 0, st>>>(keys, n, fp, planes, pitch, occ);
    else k_compress_uni<B, C, false><<<grid, kCompressThreads, 0, st>>>(keys, n, fp, planes, pitch, occ);
}

template <int B, int... Cs>
static bool launch_uni(int c, std::integer_sequence<int, Cs...>, const uint8_t* keys, uint64_t n,
                       const FixedPlan<B / 4>& fp, uint32_t* planes, uint64_t pitch, int grid, cudaStream_t st,
                       uint32_t* occ) {
    return ((c == Cs + 1 ? (launch_uni_c<B, Cs + 1>(keys, n, fp, planes, pitch, grid, st, occ), true) : false) || ...);
}

// Row-list variant for B in {32, 64} (a7: P_D from the key rows in sorted order): the random
// rows are loaded cooperatively, B/16 lanes per row with one 16-byte load each, into a
// shared-memory tile of 256 rows (odd 16-byte row stride), then each thread compresses its
// own row from there. A thread loading its whole row itself (k_compress_fixed<B, 4>) issues
// B/16 requests per row that each touch one sector of 32 rows: measured 1.8x slower on
// random 64-byte rows (scripts/mb_gather.cu: 0.85 vs 1.56 ms for 30 M rows).
template <int B>
__global__ void __launch_bounds__(kCompressThreads)
k_compress_rows(const uint8_t* __restrict__ keys, uint64_t n, const __grid_constant__ FixedPlan<B / 4> plan,
                uint32_t* __restrict__ planes, uint64_t pitch, uint32_t np, uint32_t toppad,
                const uint32_t* __restrict__ rows) {
    constexpr int NW = B / 4, U = B / 16, S16 = U | 1, RPI = kCompressThreads / U;   // rows per load step
    __shared__ int4 s_tile[kCompressThreads * S16];
    const uint32_t u = threadIdx.x % U, r0 = threadIdx.x / U;
    const uint64_t ntiles = (n + kCompressThreads - 1) / kCompressThreads;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t k0 = tile * kCompressThreads;
        int4 v[U];
#pragma unroll
        for (int j = 0; j < U; j++) {                     // all U loads in flight before any store
            const uint64_t i = k0 + r0 + (uint64_t)j * RPI;
            if (i < n) v[j] = ld_stream16c(keys + (uint64_t)__ldg(rows + i) * B + 16 * u);
        }
#pragma unroll
        for (int j = 0; j < U; j++)
            if (k0 + r0 + (uint64_t)j * RPI < n) s_tile[(r0 + j * RPI) * S16 + u] = v[j];
        __syncthreads();
        const uint64_t i = k0 + threadIdx.x;
        if (i < n) {
            uint32_t w[NW];
            const int4* row = s_tile + threadIdx.x * S16;
#pragma unroll
            for (int t = 0; t < U; t++) {
                const int4 x = row[t];
                w[4 * t + 0] = (uint32_t)x.x;
                w[4 * t + 1] = (uint32_t)x.y;
                w[4 * t + 2] = (uint32_t)x.z;
                w[4 * t + 3] = (uint32_t)x.w;
            }
            unsigned long long acc = 0;                      // pending bits, left-aligned
            uint32_t accbits = toppad, q = np - 1;
#pragma unroll
            for (int k = 0; k < NW; k++) {                   // most significant end of P first
                if (plan.mask[k] == 0) continue;
                uint32_t x = bswap32(w[k]) & plan.mask[k];
#pragma unroll
                for (int s = 0; s < 5; s++) x = mad_u32(x & plan.mv[k][s], (1u << (1u << s)) - 1u, x);
                acc |= ((unsigned long long)x << 32) >> accbits;
                accbits += plan.cnt[k];
                if (accbits >= 32) {
                    planes[(uint64_t)q * pitch + i] = (uint32_t)(acc >> 32);
                    acc <<= 32;
                    accbits -= 32;
                    q--;
                }
            }
            if (accbits) planes[(uint64_t)q * pitch + i] = (uint32_t)(acc >> 32);
        }
        __syncthreads();
    }
}

template <int B>
static void launch_fixed(const uint8_t* keys, uint64_t n, const GatherPlan* hplan, uint32_t* planes, uint64_t pitch,
                         uint32_t np, uint32_t lead, const uint32_t* rows, int grid, cudaStream_t st, uint32_t* occ) {
    FixedPlan<B / 4> fp;
    memset(&fp, 0, sizeof(fp));
    for (uint32_t s = 0; s < hplan->nsteps; s++) {
        const GatherStep& g = hplan->step[s];
        fp.mask[g.src] = g.mask;
        move_masks_left(g.mask, fp.mv[g.src]);
        fp.cnt[g.src] = g.cnt;
    }
    const uint32_t toppad = np * 32 - hplan->out_bits - lead;
    // rows: random key rows behind a dependent load -> 4 keys in flight per thread; in order:
    // ALU-bound, one key per thread measured fastest
    if constexpr (B >= 32) {
        if (rows) {
            k_compress_rows<B><<<grid, kCompressThreads, 0, st>>>(keys, n, fp, planes, pitch, np, toppad, rows);
            return;
        }
    }
    if constexpr (B == 32) {
        // every word holds the same number of mask bits and P_M is left-aligned: the
        // compile-time layout (k_compress_uni)
        bool uni = !rows && toppad == 0 && fp.cnt[0] > 0;
        for (int k = 1; k < B / 4 && uni; k++) uni = fp.cnt[k] == fp.cnt[0];
        if (uni && launch_uni<B>((int)fp.cnt[0], std::make_integer_sequence<int, 32>{}, keys, n, fp, planes, pitch,
                                 grid, st, occ))
            return;
    }
    if (rows) k_compress_fixed<B, 4><<<grid, kCompressThreads, 0, st>>>(keys, n, fp, planes, pitch, np, toppad, rows);
    else if (occ) k_compress_occ<B><<<grid, kCompressThreads, 0, st>>>(keys, n, fp, planes, pitch, np, toppad, occ);
    else k_compress_fixed<B, 1><<<grid, kCompressThreads, 0, st>>>(keys, n, fp, planes, pitch, np, toppad, rows);
}

static int grid_for(uint64_t work, int per_sm, int sms) {
    uint64_t want = (work + 255) / 256;
    uint64_t cap = (uint64_t)sms * per_sm;
    if (want == 0) want = 1;
    return (int)(want < cap ? want : cap);
}

bool compress_marks_occupancy(const uint8_t* keys, uint32_t B) {
    return ((uintptr_t)keys & 15) == 0 && (B == 8 || B == 16 || B == 32 || B == 64);
}

cudaError_t launch_compress(const uint8_t* keys, uint64_t n, uint32_t B, const GatherPlan* dplan,
                            const GatherPlan* hplan, uint32_t np, uint32_t* planes, uint64_t pitch, int sms,
                            cudaStream_t st, uint32_t lead, const uint32_t* rows, uint32_t* occ) {
    if (n == 0 || np == 0) return cudaSuccess;
    const uint32_t nsteps = hplan->nsteps;
    if (compress_marks_occupancy(keys, B)) {
        int grid = grid_for(n, 8, sms);
        switch (B) {
            case 8: launch_fixed<8>(keys, n, hplan, planes, pitch, np, lead, rows, grid, st, occ); break;
            case 16: launch_fixed<16>(keys, n, hplan, planes, pitch, np, lead, rows, grid, st, occ); break;
            case 32: launch_fixed<32>(keys, n, hplan, planes, pitch, np, lead, rows, grid, st, occ); break;
            default: launch_fixed<64>(keys, n, hplan, planes, pitch, np, lead, rows, grid, st, occ); break;
        }
        return cudaGetLastError();
    }
    if (occ) return cudaErrorInvalidValue;                       // (occupancy marking: fixed widths only)
    if ((B & 15) == 0 && ((uintptr_t)keys & 15) == 0 && !rows) {
        uint32_t S16 = (B >> 4) | 1;
        size_t smem = (size_t)kCompressThreads * S16 * 16;
        raise_smem_limit((const void*)k_compress_tiled, smem);
        int per_sm = smem <= 24 * 1024 ? 8 : smem <= 48 * 1024 ? 4 : smem <= 100 * 1024 ? 2 : 1;
        k_compress_tiled<<<grid_for(n, per_sm, sms), kCompressThreads, smem, st>>>(keys, n, B, dplan, nsteps,
                                                                                   np, planes, pitch, lead);
    } else {
        k_compress_generic<<<grid_for(n, 8, sms), kCompressThreads, 0, st>>>(keys, n, B, dplan, nsteps, np,
                                                                             planes, pitch, lead, rows);
    }
    return cudaGetLastError();
}

cudaError_t launch_repack(const uint32_t* in, uint64_t in_pitch, uint64_t n, const GatherPlan* dplan,
                          uint32_t nsteps, uint32_t np, uint32_t* out, uint64_t out_pitch, int sms,
                          cudaStream_t st, const uint32_t* rows) {
    if (n == 0 || np == 0) return cudaSuccess;
    k_repack<<<grid_for(n, 8, sms), kCompressThreads, 0, st>>>(in, in_pitch, n, dplan, nsteps, np, out,
                                                               out_pitch, rows);
    return cudaGetLastError();
}

}  // namespace cks

// k_mask.cu -- a1: superset of the distinction bits in one pass over the keys.
//
// Per byte position j we record which of the 256 byte values occur (a 256-bit
// occupancy set). From it:
//   D+_j = D-bits of the sorted distinct occurring values (Theorem 1, applied to
//          the byte values; reading R2) -- a superset of D,
//   V_j  = bits that are 1 in some occurring value and 0 in another
//        = OR over keys of (key XOR key_0) restricted to byte j.
// Layout: keys u8[n][B] row-major; occupancy u32[B][8] in global memory, bit (v & 31) of
// word [j][v >> 5] set when value v occurs at byte j. In shared memory each position's 8
// words are padded to a stride of 9 so that positions 16 apart (read by the two halves of
// a warp when B = 32) fall in different banks.
#include "cks_internal.h"
#include "k_occ_flags.cuh"

namespace cks {

__device__ __forceinline__ int4 ld_stream16(const void* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// Test-before-set: occupancy saturates after a few keys, so almost every byte costs
// one shared-memory load and no atomic.
__device__ __forceinline__ void occ_mark(uint32_t* occ, uint32_t j, uint32_t v) {
    uint32_t w = j * 9 + (v >> 5), bit = 1u << (v & 31);
    if (!(occ[w] & bit)) atomicOr(&occ[w], bit);
}

__device__ __forceinline__ void occ_word(uint32_t* occ, uint32_t j0, uint32_t Bm1, uint32_t x) {
#pragma unroll
    for (int b = 0; b < 4; b++) occ_mark(occ, (j0 + b) & Bm1, (x >> (8 * b)) & 0xFF);
}

// Fast path: B is a power of two and the key array is 16-byte aligned. Every 16-byte
// chunk then starts at byte position (16c) mod B and covers positions j0..j0+15 (mod B).
__global__ void __launch_bounds__(256) k_occupancy_pow2(const uint8_t* __restrict__ keys,
                                                        uint64_t total, uint32_t B,
                                                        uint32_t* __restrict__ occ_g) {
    extern __shared__ uint32_t occ[];
    for (uint32_t i = threadIdx.x; i < B * 9; i += blockDim.x) occ[i] = 0;
    __syncthreads();
    const uint32_t Bm1 = B - 1;
    const uint64_t nchunks = total >> 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    constexpr int U = 4;
    uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; c + (U - 1) * stride < nchunks; c += U * stride) {
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; u++) v[u] = ld_stream16(keys + ((c + u * stride) << 4));
#pragma unroll
        for (int u = 0; u < U; u++) {
            uint32_t j0 = (uint32_t)(((c + u * stride) << 4) & Bm1);
            occ_word(occ, j0 + 0, Bm1, (uint32_t)v[u].x);
            occ_word(occ, j0 + 4, Bm1, (uint32_t)v[u].y);
            occ_word(occ, j0 + 8, Bm1, (uint32_t)v[u].z);
            occ_word(occ, j0 + 12, Bm1, (uint32_t)v[u].w);
        }
    }
    for (; c < nchunks; c += stride) {
        int4 v = ld_stream16(keys + (c << 4));
        uint32_t j0 = (uint32_t)((c << 4) & Bm1);
        occ_word(occ, j0 + 0, Bm1, (uint32_t)v.x);
        occ_word(occ, j0 + 4, Bm1, (uint32_t)v.y);
        occ_word(occ, j0 + 8, Bm1, (uint32_t)v.z);
        occ_word(occ, j0 + 12, Bm1, (uint32_t)v.w);
    }
    if (blockIdx.x == 0) {                                   // ragged tail (< 16 bytes)
        for (uint64_t f = (nchunks << 4) + threadIdx.x; f < total; f += blockDim.x)
            occ_mark(occ, (uint32_t)(f & Bm1), keys[f]);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < B * 8; i += blockDim.x) {
        uint32_t v = occ[(i >> 3) * 9 + (i & 7)];
        if (v) atomicOr(&occ_g[i], v);
    }
}

// Generic path (any B, any alignment): thread per key, byte loads.
__global__ void __launch_bounds__(256) k_occupancy_generic(const uint8_t* __restrict__ keys,
                                                           uint64_t n, uint32_t B,
                                                           uint32_t* __restrict__ occ_g) {
    extern __shared__ uint32_t occ[];
    for (uint32_t i = threadIdx.x; i < B * 9; i += blockDim.x) occ[i] = 0;
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint8_t* k = keys + i * B;
        for (uint32_t j = 0; j < B; j++) occ_mark(occ, j, k[j]);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < B * 8; i += blockDim.x) {
        uint32_t v = occ[(i >> 3) * 9 + (i & 7)];
        if (v) atomicOr(&occ_g[i], v);
    }
}

// One thread per byte position: walk the occurring values in increasing order and
// set the D-bit (leading differing bit) of each adjacent pair.
__global__ void k_occ_finalize(const uint32_t* __restrict__ occ, uint32_t B, uint64_t n,
                               uint8_t* __restrict__ dplus, uint8_t* __restrict__ variant) {
    for (uint32_t j = threadIdx.x; j < B; j += blockDim.x) {
        uint32_t dp = 0, vor = 0, vand = 0xFF;
        int prev = -1;
        for (int w = 0; w < 8; w++) {
            uint32_t bits = occ[j * 8 + w];
            while (bits) {
                int v = w * 32 + __ffs(bits) - 1;
                bits &= bits - 1;
                if (prev >= 0) dp |= 0x80u >> (__clz((uint32_t)(prev ^ v)) - 24);
                vor |= (uint32_t)v;
                vand &= (uint32_t)v;
                prev = v;
            }
        }
        dplus[j] = (uint8_t)dp;
        variant[j] = (n > 0) ? (uint8_t)(vor & ~vand) : 0;
    }
}

// Specialised paths for a compile-time key width B in {8, 16} (chunk per thread, below) and
// {32, 64} (key per thread, k_occupancy_rows), 16-byte aligned keys.
// Occupancy is kept as one flag BYTE per (position, value) in shared memory, so marking a
// byte is a plain store of 1 -- no load, no test, no atomic (every writer stores the same
// value): extract the byte (PRMT), add it to the position's row, store. Rows are padded by 4
// bytes so that rows start in different banks.
// Each thread keeps U 16-byte chunks in flight. The flags are folded into the u32 bitsets
// at the end.
template <int B>
__global__ void __launch_bounds__(256) k_occupancy_bytes(const uint8_t* __restrict__ keys, uint64_t nchunks,
                                                         uint32_t* __restrict__ occ_g) {
    __shared__ __align__(16) uint8_t flag[B * kRowBytes];
    for (uint32_t i = threadIdx.x; i < B * kRowBytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(flag)[i] = 0;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    constexpr int U = 4;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += U * stride) {
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; u++)
            v[u] = (c + u * stride < nchunks) ? ld_stream16(keys + ((c + u * stride) << 4)) : make_int4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (c + u * stride >= nchunks) break;
            const uint32_t j0 = B > 16 ? (uint32_t)(((c + u * stride) << 4) & (B - 1)) : 0u;
            uint8_t* row = flag + j0 * kRowBytes;
            const uint32_t w[4] = {(uint32_t)v[u].x, (uint32_t)v[u].y, (uint32_t)v[u].z, (uint32_t)v[u].w};
#pragma unroll
            for (int b = 0; b < 16; b++) {
                const int jr = B >= 16 ? b : (b & (B - 1));
                const uint32_t val = __byte_perm(w[b >> 2], 0, 0x4440 + (b & 3));
                row[jr * kRowBytes + val] = 1;
            }
        }
    }
    __syncthreads();
    fold_flags<B>(flag, occ_g);
}

// B in {32, 64}: thread per key. In the chunk-per-thread kernel above the lanes of a warp
// hold chunks of B/16 different byte positions, so one store instruction hits B/16 flag rows
// at the same value offsets -- B/16-way bank conflicts on text keys, whose bytes span few
// banks. Here every lane of a store instruction marks the same position j of its own key:
// one row, values in distinct words (or the same word), conflict-free. The key's 16-byte
// loads are L1-allocating so the lanes' 64-byte-strided loads fetch each sector once.
template <int B>
__global__ void __launch_bounds__(256) k_occupancy_rows(const uint8_t* __restrict__ keys, uint64_t n,
                                                        uint32_t* __restrict__ occ_g) {
    __shared__ __align__(16) uint8_t flag[B * kRowBytes];
    for (uint32_t i = threadIdx.x; i < B * kRowBytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(flag)[i] = 0;
    __syncthreads();
    constexpr int U = B / 16;                                 // 16-byte units per key
    constexpr int KPT = 128 / B;                              // keys in flight per thread
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += KPT * stride) {
        int4 v[KPT][U];
#pragma unroll
        for (int k = 0; k < KPT; k++)
#pragma unroll
            for (int u = 0; u < U; u++)
                v[k][u] = i + k * stride < n ? __ldg(reinterpret_cast<const int4*>(keys + (i + k * stride) * B) + u)
                                             : make_int4(0, 0, 0, 0);
#pragma unroll
        for (int k = 0; k < KPT; k++) {
            if (i + k * stride >= n) break;
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t w[4] = {(uint32_t)v[k][u].x, (uint32_t)v[k][u].y, (uint32_t)v[k][u].z,
                                       (uint32_t)v[k][u].w};
#pragma unroll
                for (int b = 0; b < 16; b++)
                    flag[(16 * u + b) * kRowBytes + __byte_perm(w[b >> 2], 0, 0x4440 + (b & 3))] = 1;
            }
        }
    }
    __syncthreads();
    fold_flags<B>(flag, occ_g);
}

cudaError_t launch_occupancy(const uint8_t* keys, uint64_t n, uint32_t B, uint32_t* occ,
                             int sms, cudaStream_t st) {
    size_t smem = (size_t)B * 9 * sizeof(uint32_t);
    bool pow2 = (B & (B - 1)) == 0;
    bool aligned = ((uintptr_t)keys & 15) == 0;
    if (aligned && (B == 32 || B == 64)) {
        uint64_t want = (n + 255) / 256;
        int grid = (int)(want < (uint64_t)sms * 8 ? (want ? want : 1) : (uint64_t)sms * 8);
        if (B == 32) k_occupancy_rows<32><<<grid, 256, 0, st>>>(keys, n, occ);
        else k_occupancy_rows<64><<<grid, 256, 0, st>>>(keys, n, occ);
    } else if (aligned && (B == 8 || B == 16) && ((n * B) & 15) == 0) {
        uint64_t nchunks = (n * B) >> 4;
        uint64_t want = (nchunks + 255) / 256;
        int grid = (int)(want < (uint64_t)sms * 8 ? (want ? want : 1) : (uint64_t)sms * 8);
        switch (B) {
            case 8: k_occupancy_bytes<8><<<grid, 256, 0, st>>>(keys, nchunks, occ); break;
            default: k_occupancy_bytes<16><<<grid, 256, 0, st>>>(keys, nchunks, occ); break;
        }
    } else if (pow2 && aligned) {
        uint64_t nchunks = (n * B) >> 4;
        uint64_t want = (nchunks + 255) / 256;
        int grid = (int)(want < (uint64_t)sms * 8 ? (want ? want : 1) : (uint64_t)sms * 8);
        k_occupancy_pow2<<<grid, 256, smem, st>>>(keys, n * B, B, occ);
    } else {
        uint64_t want = (n + 255) / 256;
        int grid = (int)(want < (uint64_t)sms * 8 ? (want ? want : 1) : (uint64_t)sms * 8);
        raise_smem_limit((const void*)k_occupancy_generic, smem);
        k_occupancy_generic<<<grid, 256, smem, st>>>(keys, n, B, occ);
    }
    return cudaGetLastError();
}

// Occupancy of a strided sample of rows (thread per sampled row, B in {8, 16, 32, 64}, 16-byte
// aligned keys): the speculative first build's mask (cks_api.cu build_common). Row i*step for
// i < samples.
template <int B>
__global__ void __launch_bounds__(256) k_occupancy_sample(const uint8_t* __restrict__ keys, uint64_t step,
                                                          uint32_t samples, uint32_t* __restrict__ occ_g) {
    __shared__ __align__(16) uint8_t flag[B * kRowBytes];
    for (uint32_t i = threadIdx.x; i < B * kRowBytes / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(flag)[i] = 0;
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < samples; i += gridDim.x * blockDim.x) {
        const uint8_t* row = keys + (uint64_t)i * step * B;
#pragma unroll
        for (int u = 0; u < (B >= 16 ? B / 16 : 1); u++) {
            uint32_t w[4];
            if (B >= 16) {
                const int4 v = __ldg(reinterpret_cast<const int4*>(row) + u);
                w[0] = (uint32_t)v.x; w[1] = (uint32_t)v.y; w[2] = (uint32_t)v.z; w[3] = (uint32_t)v.w;
            } else {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(row));
                w[0] = v.x; w[1] = v.y; w[2] = 0; w[3] = 0;
            }
#pragma unroll
            for (int b = 0; b < (B >= 16 ? 16 : B); b++)
                flag[(16 * u + b) * kRowBytes + __byte_perm(w[b >> 2], 0, 0x4440 + (b & 3))] = 1;
        }
    }
    __syncthreads();
    fold_flags<B>(flag, occ_g);
}

cudaError_t launch_occupancy_sample(const uint8_t* keys, uint64_t n, uint32_t B, uint32_t samples, uint32_t* occ,
                                    cudaStream_t st) {
    if (n == 0 || samples == 0) return cudaSuccess;
    const uint64_t step = n / samples ? n / samples : 1;
    const uint32_t cnt = (uint32_t)(n / step < samples ? n / step : samples);
    const unsigned grid = (cnt + 255) / 256 < 64 ? (cnt + 255) / 256 : 64;
    switch (B) {
        case 8: k_occupancy_sample<8><<<grid, 256, 0, st>>>(keys, step, cnt, occ); break;
        case 16: k_occupancy_sample<16><<<grid, 256, 0, st>>>(keys, step, cnt, occ); break;
        case 32: k_occupancy_sample<32><<<grid, 256, 0, st>>>(keys, step, cnt, occ); break;
        case 64: k_occupancy_sample<64><<<grid, 256, 0, st>>>(keys, step, cnt, occ); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_occ_finalize(const uint32_t* occ, uint32_t B, uint64_t n, uint8_t* dplus,
                                uint8_t* variant, cudaStream_t st) {
    k_occ_finalize<<<1, 256, 0, st>>>(occ, B, n, dplus, variant);
    return cudaGetLastError();
}

}  // namespace cks

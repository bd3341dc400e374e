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

// Specialised path for a compile-time key width B in {8, 16, 32, 64} (16-byte aligned
// keys): each 16-byte chunk covers byte positions j0 + 0..15 (j0 = 16c mod B, 0 for B <= 16),
// so every byte's occupancy word is a compile-time offset from one row pointer; the
// test-before-set is one shared load, one test and one predicated shared reduction (no
// branch). Loads of U chunks are issued before any test.
__device__ __forceinline__ void red_or_if(uint32_t* p, uint32_t bit, uint32_t cur) {
    asm volatile("{\n .reg .pred q;\n setp.eq.u32 q, %2, 0;\n @q red.shared.or.b32 [%0], %1;\n}"
                 ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(bit), "r"(cur & bit) : "memory");
}

template <int B>
__global__ void __launch_bounds__(256) k_occupancy_fixed(const uint8_t* __restrict__ keys, uint64_t nchunks,
                                                         uint32_t* __restrict__ occ_g) {
    __shared__ uint32_t occ[B * 9];
    for (uint32_t i = threadIdx.x; i < B * 9; i += blockDim.x) occ[i] = 0;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    constexpr int U = 2;
    for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += U * stride) {
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; u++)
            v[u] = (c + u * stride < nchunks) ? ld_stream16(keys + ((c + u * stride) << 4)) : make_int4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (c + u * stride >= nchunks) break;
            const uint32_t j0 = B > 16 ? (uint32_t)(((c + u * stride) << 4) & (B - 1)) : 0u;
            uint32_t* row = occ + j0 * 9;
            const uint32_t w[4] = {(uint32_t)v[u].x, (uint32_t)v[u].y, (uint32_t)v[u].z, (uint32_t)v[u].w};
            uint32_t* ptr[16];
            uint32_t bit[16], cur[16];
#pragma unroll
            for (int b = 0; b < 16; b++) {
                const uint32_t x = w[b >> 2] >> (8 * (b & 3));
                const int jr = B >= 16 ? b : (b & (B - 1));
                ptr[b] = row + jr * 9 + ((x >> 5) & 7);
                bit[b] = 1u << (x & 31);
            }
#pragma unroll
            for (int b = 0; b < 16; b++) cur[b] = *ptr[b];
#pragma unroll
            for (int b = 0; b < 16; b++) red_or_if(ptr[b], bit[b], cur[b]);
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < B * 8; i += blockDim.x) {
        uint32_t x = occ[(i >> 3) * 9 + (i & 7)];
        if (x) atomicOr(&occ_g[i], x);
    }
}

cudaError_t launch_occupancy(const uint8_t* keys, uint64_t n, uint32_t B, uint32_t* occ,
                             int sms, cudaStream_t st) {
    size_t smem = (size_t)B * 9 * sizeof(uint32_t);
    bool pow2 = (B & (B - 1)) == 0;
    bool aligned = ((uintptr_t)keys & 15) == 0;
    if (aligned && (B == 8 || B == 16 || B == 32 || B == 64) && ((n * B) & 15) == 0) {
        uint64_t nchunks = (n * B) >> 4;
        uint64_t want = (nchunks + 255) / 256;
        int grid = (int)(want < (uint64_t)sms * 8 ? (want ? want : 1) : (uint64_t)sms * 8);
        switch (B) {
            case 8: k_occupancy_fixed<8><<<grid, 256, 0, st>>>(keys, nchunks, occ); break;
            case 16: k_occupancy_fixed<16><<<grid, 256, 0, st>>>(keys, nchunks, occ); break;
            case 32: k_occupancy_fixed<32><<<grid, 256, 0, st>>>(keys, nchunks, occ); break;
            default: k_occupancy_fixed<64><<<grid, 256, 0, st>>>(keys, nchunks, occ); break;
        }
    } else if (pow2 && aligned) {
        uint64_t nchunks = (n * B) >> 4;
        uint64_t want = (nchunks + 255) / 256;
        int grid = (int)(want < (uint64_t)sms * 8 ? (want ? want : 1) : (uint64_t)sms * 8);
        k_occupancy_pow2<<<grid, 256, smem, st>>>(keys, n * B, B, occ);
    } else {
        uint64_t want = (n + 255) / 256;
        int grid = (int)(want < (uint64_t)sms * 8 ? (want ? want : 1) : (uint64_t)sms * 8);
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_occupancy_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_occupancy_generic<<<grid, 256, smem, st>>>(keys, n, B, occ);
    }
    return cudaGetLastError();
}

cudaError_t launch_occ_finalize(const uint32_t* occ, uint32_t B, uint64_t n, uint8_t* dplus,
                                uint8_t* variant, cudaStream_t st) {
    k_occ_finalize<<<1, 256, 0, st>>>(occ, B, n, dplus, variant);
    return cudaGetLastError();
}

}  // namespace cks

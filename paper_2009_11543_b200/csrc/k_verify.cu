// k_verify.cu -- order check of a returned permutation against the key rows.
//
// Theorem 2 makes the compressed order equal to the full-key order only when the
// sort mask contains every distinction bit (extended positions). A rebuild extracts with
// the CURRENT D-bitmap; if that mask is stale (a key was inserted since, so some
// pair's D-bit is missing from it) the compressed sort silently mis-orders keys. The check
// here is complete: a sequence is sorted by (key, row id) iff every adjacent pair is, and the
// (key, row id) order is total, so "no adjacent pair out of order" means the permutation is
// exactly the full-key order. One thread per sorted position i >= 1 compares the rows
// perm[i-1] and perm[i] (big-endian words, memcmp order) and, on a key tie, their row ids.
// Cost: one random row gather per key (plus the neighbour's row, mostly an L1/L2 hit).
#include "cks_internal.h"

namespace cks {

namespace {

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0u, 0x0123u); }

// -1 / 0 / +1: row a vs row b in memcmp order
template <int VEC>
__device__ __forceinline__ int cmp_rows(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, uint32_t B) {
    if (VEC == 16) {
        const uint4* x = reinterpret_cast<const uint4*>(a);
        const uint4* y = reinterpret_cast<const uint4*>(b);
        for (uint32_t k = 0; k < B / 16; k++) {
            const uint4 u = __ldg(x + k), v = __ldg(y + k);
            const uint32_t uu[4] = {u.x, u.y, u.z, u.w}, vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; j++)
                if (uu[j] != vv[j]) return bswap32(uu[j]) < bswap32(vv[j]) ? -1 : 1;
        }
        return 0;
    } else if (VEC == 4) {
        const uint32_t* x = reinterpret_cast<const uint32_t*>(a);
        const uint32_t* y = reinterpret_cast<const uint32_t*>(b);
        for (uint32_t k = 0; k < B / 4; k++) {
            const uint32_t u = __ldg(x + k), v = __ldg(y + k);
            if (u != v) return bswap32(u) < bswap32(v) ? -1 : 1;
        }
        return 0;
    } else {
        for (uint32_t k = 0; k < B; k++) {
            const uint8_t u = __ldg(a + k), v = __ldg(b + k);
            if (u != v) return u < v ? -1 : 1;
        }
        return 0;
    }
}

template <int VEC>
__global__ void __launch_bounds__(256)
k_verify_order(const uint8_t* __restrict__ keys, uint32_t B, const uint32_t* __restrict__ perm, uint64_t n,
               unsigned long long* __restrict__ first_bad) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t ra = __ldg(perm + i - 1), rb = __ldg(perm + i);
        const int c = cmp_rows<VEC>(keys + (uint64_t)ra * B, keys + (uint64_t)rb * B, B);
        if (c > 0 || (c == 0 && ra >= rb)) atomicMin(first_bad, (unsigned long long)i);
    }
}

}  // namespace

cudaError_t launch_verify_order(const uint8_t* keys, uint32_t B, const uint32_t* perm, uint64_t n,
                                unsigned long long* first_bad, int sms, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(first_bad, 0xFF, sizeof(unsigned long long), st);
    if (e != cudaSuccess || n < 2) return e;
    uint64_t g = (n + 255) / 256;
    const uint64_t cap = (uint64_t)sms * 8;
    if (g > cap) g = cap;
    const bool al16 = ((uintptr_t)keys & 15) == 0 && B % 16 == 0;
    const bool al4 = ((uintptr_t)keys & 3) == 0 && B % 4 == 0;
    if (al16) k_verify_order<16><<<(unsigned)g, 256, 0, st>>>(keys, B, perm, n, first_bad);
    else if (al4) k_verify_order<4><<<(unsigned)g, 256, 0, st>>>(keys, B, perm, n, first_bad);
    else k_verify_order<1><<<(unsigned)g, 256, 0, st>>>(keys, B, perm, n, first_bad);
    return cudaGetLastError();
}

}  // namespace cks

// k_occ_flags.cuh -- byte-occupancy flags shared by the superset pass (k_mask.cu) and the
// compress that marks them on the way (k_compress.cu, the speculative first build):
// one flag BYTE per (position, value) in shared memory, rows of 256 values padded by 4
// bytes so that rows start in different banks; folded into u32[B][8] bitsets at the end.
#pragma once
#include <cstdint>

namespace cks {

constexpr int kRowBytes = 260;

// fold: thread per (position, word): 32 flags -> one u32, OR-ed into the global bitsets
template <int B>
__device__ __forceinline__ void fold_flags(const uint8_t* flag, uint32_t* __restrict__ occ_g) {
    for (uint32_t i = threadIdx.x; i < B * 8; i += blockDim.x) {
        const uint8_t* f = flag + (i >> 3) * kRowBytes + (i & 7) * 32;
        uint32_t bits = 0;
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
            uint32_t q = *reinterpret_cast<const uint32_t*>(f + k);
            bits |= ((q & 0xFF) ? 1u : 0u) << k;
            bits |= ((q & 0xFF00) ? 1u : 0u) << (k + 1);
            bits |= ((q & 0xFF0000) ? 1u : 0u) << (k + 2);
            bits |= ((q & 0xFF000000) ? 1u : 0u) << (k + 3);
        }
        if (bits) atomicOr(&occ_g[i], bits);
    }
}

}  // namespace cks

// k_adjacent.cu -- a6: distinction bits of sorted-adjacent keys and
// a8: bottom-up bulk load (Sec. 5.3).
//
// a6: for sorted compressed keys P_{i-1}, P_i the first differing compressed bit is the
// highest set bit of P_{i-1} XOR P_i; counted from the most significant end it indexes
// the D-offset table of the sort mask, D_i = D-offset[D-bit(Compress, Compress)].
// The union of the D_i is the exact D (Theorem 1), a subset of the sort mask
// (P:411). Layout: planes u32[np][n]; D accumulated as u32 words where bit (31 - p%32) of
// word p/32 is key position p (so the words, read big-endian, are the mask bytes).
#include "cks_internal.h"

namespace cks {

__global__ void __launch_bounds__(256)
k_adjacent(const uint32_t* __restrict__ planes, uint64_t pitch, uint64_t n, uint32_t m, uint32_t np,
           const uint16_t* __restrict__ moff, uint32_t nwords, uint16_t* __restrict__ dbit,
           uint32_t* __restrict__ dacc) {
    extern __shared__ uint32_t s_dyn[];
    uint32_t* s_bm = s_dyn;                                      // [nwords]
    uint16_t* s_moff = reinterpret_cast<uint16_t*>(s_dyn + nwords); // [m]
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x) s_bm[w] = 0;
    for (uint32_t t = threadIdx.x; t < m; t += blockDim.x) s_moff[t] = moff[t];
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t d = CKS_NONE_INTERNAL;
        if (i > 0) {
            for (int q = (int)np - 1; q >= 0; q--) {
                uint32_t x = planes[(uint64_t)q * pitch + i] ^ planes[(uint64_t)q * pitch + i - 1];
                if (x) {
                    uint32_t bitpos = 32u * (uint32_t)q + 31u - (uint32_t)__clz(x);   // bit of P
                    uint32_t t = (m - 1) - bitpos;                                  // compressed position
                    d = s_moff[t];
                    uint32_t w = d >> 5, b = 0x80000000u >> (d & 31);
                    if (!(s_bm[w] & b)) atomicOr(&s_bm[w], b);
                    break;
                }
            }
        }
        if (dbit) dbit[i] = (uint16_t)d;
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x)
        if (s_bm[w]) atomicOr(&dacc[w], s_bm[w]);
}

cudaError_t launch_adjacent(const uint32_t* planes, uint64_t pitch, uint64_t n, uint32_t m, const uint16_t* moff,
                            uint32_t B, uint16_t* dbit, uint32_t* dacc, int sms, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    uint32_t np = (m + 31) / 32;
    uint32_t nwords = (8 * B + 31) / 32;
    size_t smem = (size_t)nwords * 4 + (size_t)m * 2;
    uint64_t want = (n + 255) / 256;
    int grid = (int)(want < (uint64_t)sms * 8 ? want : (uint64_t)sms * 8);
    k_adjacent<<<grid, 256, smem, st>>>(planes, pitch, n, m, np, moff, nwords, dbit, dacc);
    return cudaGetLastError();
}

__global__ void k_iota(uint32_t* out, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)i;
}
__global__ void k_fill_u16(uint16_t* out, uint64_t n, uint16_t v) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = v;
}
cudaError_t launch_iota(uint32_t* out, uint64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    uint64_t want = (n + 255) / 256;
    k_iota<<<(unsigned)(want < 4096 ? want : 4096), 256, 0, st>>>(out, n);
    return cudaGetLastError();
}
cudaError_t launch_fill_u16(uint16_t* out, uint64_t n, uint16_t v, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    uint64_t want = (n + 255) / 256;
    k_fill_u16<<<(unsigned)(want < 4096 ? want : 4096), 256, 0, st>>>(out, n, v);
    return cudaGetLastError();
}

// ---- a8 bulk load ------------------------------------------------------------------------
// Leaves: slot e of leaf j holds sorted entry x = j*per + e (e < per). Inner level l: slot
// e of node j holds entry x = j*per + e whose child is node x of level l-1; its key is the
// highest key under that child, sorted index hi = min((x+1)*span, n) - 1. The
// entry D-bit against the previous entry's highest key is the minimum of D_k over the
// keys it adds, (x*span, hi] (Lemma 1), carried level to level as rmin.

__global__ void k_bulk_leaves(const uint32_t* __restrict__ perm, const uint16_t* __restrict__ dbit,
                              BulkLevel L, uint32_t fanout, uint32_t per, uint32_t* __restrict__ node_cnt,
                              uint32_t* __restrict__ rid, uint16_t* __restrict__ edbit) {
    // slots < 2^32 (n < 2^32 and per >= fanout/2 in practice): 32-bit index arithmetic
    const uint32_t slots = (uint32_t)(L.nodes * fanout);
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < slots; s += gridDim.x * blockDim.x) {
        uint32_t j = s / fanout;
        uint32_t e = s - j * fanout;
        uint64_t x = (uint64_t)j * per + e;
        bool ok = e < per && x < L.entries;
        rid[s] = ok ? perm[x] : 0xFFFFFFFFu;
        if (edbit) edbit[s] = ok ? dbit[x] : (uint16_t)CKS_NONE_INTERNAL;
        if (e == 0) {
            uint64_t rem = L.entries - (uint64_t)j * per;
            node_cnt[j] = (uint32_t)(rem < per ? rem : per);
        }
    }
}

__global__ void k_bulk_inner(const uint32_t* __restrict__ perm, const uint16_t* __restrict__ rmin_below,
                             BulkLevel L, uint64_t n, uint64_t entries_below, uint32_t fanout, uint32_t per,
                             uint32_t* __restrict__ node_cnt, uint32_t* __restrict__ rid,
                             uint16_t* __restrict__ edbit, uint32_t* __restrict__ child,
                             uint64_t inner_off, uint16_t* __restrict__ rmin) {
    const uint32_t slots = (uint32_t)(L.nodes * fanout);
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < slots; s += gridDim.x * blockDim.x) {
        uint32_t j = s / fanout;
        uint32_t e = s - j * fanout;
        uint64_t x = (uint64_t)j * per + e;
        bool ok = e < per && x < L.entries;
        uint64_t gs = (L.node_off + j) * fanout + e;                  // global slot
        uint64_t cs = (L.node_off - inner_off + j) * fanout + e;      // inner-only slot
        if (ok) {
            uint64_t hi = (x + 1) * L.span;
            hi = (hi < n ? hi : n) - 1;
            rid[gs] = perm[hi];
            if (child) child[cs] = (uint32_t)(L.below_off + x);
            if (rmin_below) {
                uint64_t y0 = x * per, y1 = y0 + per;
                if (y1 > entries_below) y1 = entries_below;
                uint32_t mn = CKS_NONE_INTERNAL;
                for (uint64_t y = y0; y < y1; y++) mn = min(mn, (uint32_t)rmin_below[y]);
                rmin[x] = (uint16_t)mn;
                if (edbit) edbit[gs] = x == 0 ? (uint16_t)CKS_NONE_INTERNAL : (uint16_t)mn;
            }
        } else {
            rid[gs] = 0xFFFFFFFFu;
            if (child) child[cs] = 0xFFFFFFFFu;
            if (edbit) edbit[gs] = (uint16_t)CKS_NONE_INTERNAL;
        }
        if (e == 0) {
            uint64_t rem = L.entries - j * per;
            node_cnt[L.node_off + j] = (uint32_t)(rem < per ? rem : per);
        }
    }
}

static unsigned grid1d(uint64_t work) {
    uint64_t want = (work + 255) / 256;
    if (want == 0) want = 1;
    return (unsigned)(want < 148 * 16 ? want : 148 * 16);
}

cudaError_t launch_bulk_leaves(const uint32_t* perm, const uint16_t* dbit, const BulkLevel& L,
                               uint32_t fanout, uint32_t per, uint32_t* node_cnt, uint32_t* rid,
                               uint16_t* edbit, uint16_t* /*rmin*/, cudaStream_t st) {
    k_bulk_leaves<<<grid1d(L.nodes * fanout), 256, 0, st>>>(perm, dbit, L, fanout, per, node_cnt, rid,
                                                            edbit);
    return cudaGetLastError();
}

cudaError_t launch_bulk_inner(const uint32_t* perm, const uint16_t* rmin_below, const BulkLevel& L,
                              uint64_t n, uint32_t fanout, uint32_t per, uint32_t* node_cnt,
                              uint32_t* rid, uint16_t* edbit, uint32_t* child, uint64_t inner_off,
                              uint16_t* rmin, cudaStream_t st) {
    // entries_below: entries of the level below = nodes of the level two below, i.e. the
    // number of children's entries; equal to L.entries * per bounded by the true count,
    // which the caller encodes as span/per keys per entry at the level below.
    uint64_t entries_below = (n + L.span / per - 1) / (L.span / per);
    k_bulk_inner<<<grid1d(L.nodes * fanout), 256, 0, st>>>(perm, rmin_below, L, n, entries_below, fanout,
                                                           per, node_cnt, rid, edbit, child, inner_off,
                                                           rmin);
    return cudaGetLastError();
}

}  // namespace cks

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
    const uint32_t lane = threadIdx.x & 31;
    constexpr int U = 4;                                         // elements per thread per step
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n + (U - 1) * stride;
         i0 += U * stride) {
        uint32_t d[U];
        uint32_t diffq[U];                                        // highest differing plane, or -1
        uint32_t x[U];
#pragma unroll
        for (int u = 0; u < U; u++) { diffq[u] = 0xFFFFFFFFu; x[u] = 0; }
        // walk planes from the most significant; the previous key comes from lane-1 (lane 0 loads it)
        for (int q = (int)np - 1; q >= 0; q--) {
            const uint32_t* pl = planes + (uint64_t)q * pitch;
            uint32_t cur[U], prv[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint64_t i = i0 + u * stride;
                cur[u] = i < n ? __ldg(pl + i) : 0u;
                prv[u] = (lane == 0 && i > 0 && i < n) ? __ldg(pl + i - 1) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                uint32_t up = __shfl_up_sync(0xffffffffu, cur[u], 1);
                if (lane) prv[u] = up;
                uint32_t xx = cur[u] ^ prv[u];
                if (diffq[u] == 0xFFFFFFFFu && xx) { diffq[u] = (uint32_t)q; x[u] = xx; }
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint64_t i = i0 + u * stride;
            d[u] = CKS_NONE_INTERNAL;
            if (i > 0 && i < n && diffq[u] != 0xFFFFFFFFu) {
                uint32_t bitpos = 32u * diffq[u] + 31u - (uint32_t)__clz(x[u]);   // bit of P
                uint32_t t = (m - 1) - bitpos;                                       // compressed position
                d[u] = s_moff[t];
                uint32_t w = d[u] >> 5, b = 0x80000000u >> (d[u] & 31);
                if (!(s_bm[w] & b)) atomicOr(&s_bm[w], b);
            }
            if (dbit && i < n) dbit[i] = (uint16_t)d[u];
        }
    }
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x)
        if (s_bm[w]) atomicOr(&dacc[w], s_bm[w]);
}

// Vectorised path (planes 16-byte aligned, pitch % 8 == 0, dbit 16-byte aligned): a thread
// owns 8 consecutive sorted keys, loads each of its planes with two 16-byte loads (all
// planes in flight at once, NP <= 4), takes the predecessor of its first key from lane - 1
// (lane 0 loads it), and writes its 8 D_i with one 16-byte store.
template <int NP>
__global__ void __launch_bounds__(256)
k_adjacent8(const uint32_t* __restrict__ planes, uint64_t pitch, uint64_t n, uint32_t m,
            const uint16_t* __restrict__ moff, uint32_t nwords, uint16_t* __restrict__ dbit,
            uint32_t* __restrict__ dacc) {
    extern __shared__ uint32_t s_dyn[];
    uint32_t* s_bm = s_dyn;
    uint16_t* s_moff = reinterpret_cast<uint16_t*>(s_dyn + nwords);
    for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x) s_bm[w] = 0;
    for (uint32_t t = threadIdx.x; t < m; t += blockDim.x) s_moff[t] = moff[t];
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t groups = (n + 7) / 8;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g0 = (uint64_t)blockIdx.x * blockDim.x; g0 < groups; g0 += stride) {
        const uint64_t g = g0 + threadIdx.x;                      // warp-uniform loop bound
        const uint64_t i0 = g * 8;
        const bool full = i0 + 8 <= n;
        uint32_t v[NP][8];
        uint32_t pv[NP];
#pragma unroll
        for (int q = 0; q < NP; q++) {
            const uint32_t* pl = planes + (uint64_t)q * pitch;
            if (full) {
                uint4 a = __ldg(reinterpret_cast<const uint4*>(pl + i0));
                uint4 b = __ldg(reinterpret_cast<const uint4*>(pl + i0 + 4));
                v[q][0] = a.x; v[q][1] = a.y; v[q][2] = a.z; v[q][3] = a.w;
                v[q][4] = b.x; v[q][5] = b.y; v[q][6] = b.z; v[q][7] = b.w;
            } else {
#pragma unroll
                for (int k = 0; k < 8; k++) v[q][k] = (g < groups && i0 + k < n) ? __ldg(pl + i0 + k) : 0u;
            }
            pv[q] = (lane == 0 && g < groups && i0 > 0) ? __ldg(pl + i0 - 1) : 0u;
        }
#pragma unroll
        for (int q = 0; q < NP; q++) {
            uint32_t up = __shfl_up_sync(0xffffffffu, v[q][7], 1);
            if (lane) pv[q] = up;
        }
        uint16_t out[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint64_t i = i0 + k;
            uint32_t d = CKS_NONE_INTERNAL;
            int hq = -1;
            uint32_t hx = 0;
#pragma unroll
            for (int q = 0; q < NP; q++) {                        // highest differing plane wins
                uint32_t x = v[q][k] ^ (k ? v[q][k - 1] : pv[q]);
                if (x) { hq = q; hx = x; }
            }
            if (g < groups && i > 0 && i < n && hq >= 0) {
                uint32_t bitpos = 32u * (uint32_t)hq + 31u - (uint32_t)__clz(hx);
                d = s_moff[(m - 1) - bitpos];
                uint32_t w = d >> 5, b = 0x80000000u >> (d & 31);
                if (!(s_bm[w] & b)) atomicOr(&s_bm[w], b);
            }
            out[k] = (uint16_t)d;
        }
        if (dbit && g < groups) {
            if (full) {
                uint4 o;
                o.x = out[0] | ((uint32_t)out[1] << 16);
                o.y = out[2] | ((uint32_t)out[3] << 16);
                o.z = out[4] | ((uint32_t)out[5] << 16);
                o.w = out[6] | ((uint32_t)out[7] << 16);
                *reinterpret_cast<uint4*>(dbit + i0) = o;
            } else {
#pragma unroll
                for (int k = 0; k < 8; k++)
                    if (i0 + k < n) dbit[i0 + k] = out[k];
            }
        }
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
    const bool vec = ((uintptr_t)planes % 16 == 0) && (pitch % 8 == 0) && ((uintptr_t)dbit % 16 == 0) && np <= 4;
    if (vec) {
        uint64_t groups = (n + 7) / 8;
        uint64_t want = (groups + 255) / 256;
        int grid = (int)(want < (uint64_t)sms * 8 ? want : (uint64_t)sms * 8);
        switch (np) {
            case 1: k_adjacent8<1><<<grid, 256, smem, st>>>(planes, pitch, n, m, moff, nwords, dbit, dacc); break;
            case 2: k_adjacent8<2><<<grid, 256, smem, st>>>(planes, pitch, n, m, moff, nwords, dbit, dacc); break;
            case 3: k_adjacent8<3><<<grid, 256, smem, st>>>(planes, pitch, n, m, moff, nwords, dbit, dacc); break;
            default: k_adjacent8<4><<<grid, 256, smem, st>>>(planes, pitch, n, m, moff, nwords, dbit, dacc); break;
        }
        return cudaGetLastError();
    }
    uint64_t want = (n + 1023) / 1024;
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
// One warp per node. Leaves: slot e of leaf j holds sorted entry x = j*per + e (e < per).
// Inner level l: slot e of node j holds entry x = j*per + e whose child is node x of level
// l-1; its key is the highest key under that child, sorted index hi = min((x+1)*span, n) - 1
// (P:356). The D-bit of an entry against the previous entry's highest key is the minimum
// of D_k over the keys the entry adds (Lemma 1) = the minimum over its child node,
// so every level also emits its nodes' minima (rmin) for the level above.

__device__ __forceinline__ uint32_t warp_min(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__global__ void __launch_bounds__(256)
k_bulk_leaves(const uint32_t* __restrict__ perm, const uint16_t* __restrict__ dbit, BulkLevel L,
              uint32_t fanout, uint32_t per, uint32_t* __restrict__ node_cnt, uint32_t* __restrict__ rid,
              uint16_t* __restrict__ edbit, uint16_t* __restrict__ rmin) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t j = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < L.nodes; j += nwarps) {
        const uint64_t x0 = j * per;
        uint32_t mn = CKS_NONE_INTERNAL;
        for (uint32_t e = lane; e < fanout; e += 32) {
            const uint64_t x = x0 + e;
            const bool ok = e < per && x < L.entries;
            const uint64_t s = j * fanout + e;
            rid[s] = ok ? perm[x] : 0xFFFFFFFFu;
            if (dbit) {
                uint32_t d = ok ? dbit[x] : CKS_NONE_INTERNAL;
                if (edbit) edbit[s] = (uint16_t)d;
                mn = min(mn, d);
            }
        }
        if (rmin) mn = warp_min(mn);
        if (lane == 0) {
            uint64_t rem = L.entries - x0;
            node_cnt[j] = (uint32_t)(rem < per ? rem : per);
            if (rmin) rmin[j] = (uint16_t)mn;
        }
    }
}

__global__ void __launch_bounds__(256)
k_bulk_inner(const uint32_t* __restrict__ perm, const uint16_t* __restrict__ rmin_below, BulkLevel L,
             uint64_t n, uint32_t fanout, uint32_t per, uint32_t* __restrict__ node_cnt,
             uint32_t* __restrict__ rid, uint16_t* __restrict__ edbit, uint32_t* __restrict__ child,
             uint64_t inner_off, uint16_t* __restrict__ rmin, int first_none) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t j = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < L.nodes; j += nwarps) {
        uint32_t mn = CKS_NONE_INTERNAL;
        for (uint32_t e = lane; e < fanout; e += 32) {
            const uint64_t x = j * per + e;
            const bool ok = e < per && x < L.entries;
            const uint64_t gs = (L.node_off + j) * fanout + e;               // global slot
            const uint64_t cs = (L.node_off - inner_off + j) * fanout + e;   // inner-only slot
            if (ok) {
                uint64_t hi = (x + 1) * L.span;
                hi = (hi < n ? hi : n) - 1;
                rid[gs] = perm[hi];
                if (child) child[cs] = (uint32_t)(L.below_off + x);
                if (rmin_below) {
                    uint32_t v = rmin_below[x];
                    mn = min(mn, v);
                    if (edbit) edbit[gs] = (x == 0 && first_none) ? (uint16_t)CKS_NONE_INTERNAL : (uint16_t)v;
                }
            } else {
                rid[gs] = 0xFFFFFFFFu;
                if (child) child[cs] = 0xFFFFFFFFu;
                if (edbit) edbit[gs] = (uint16_t)CKS_NONE_INTERNAL;
            }
        }
        if (rmin) mn = warp_min(mn);
        if (lane == 0) {
            uint64_t rem = L.entries - j * per;
            node_cnt[L.node_off + j] = (uint32_t)(rem < per ? rem : per);
            if (rmin) rmin[j] = (uint16_t)mn;
        }
    }
}

// Full leaves (per == fanout, fanout % 8 == 0, 16-byte aligned arrays): the leaf level is
// perm and dbit in order, padded; a thread copies 8 consecutive slots with 16-byte accesses
// and the fanout/8 threads of a node combine their minima with shuffles.
__global__ void __launch_bounds__(256)
k_bulk_leaves_full(const uint32_t* __restrict__ perm, const uint16_t* __restrict__ dbit, uint64_t n,
                   uint64_t nodes, uint32_t fanout, uint32_t* __restrict__ node_cnt,
                   uint32_t* __restrict__ rid, uint16_t* __restrict__ edbit, uint16_t* __restrict__ rmin) {
    const uint32_t tpn = fanout / 8;                              // threads per node (power of two <= 32)
    const uint64_t groups = nodes * tpn;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g0 = (uint64_t)blockIdx.x * blockDim.x; g0 < groups; g0 += stride) {
        const uint64_t g = g0 + threadIdx.x;
        const uint64_t x0 = g * 8;
        uint32_t mn = CKS_NONE_INTERNAL;
        if (g < groups) {
            uint4 r0, r1, dd;
            if (x0 + 8 <= n) {
                r0 = __ldg(reinterpret_cast<const uint4*>(perm + x0));
                r1 = __ldg(reinterpret_cast<const uint4*>(perm + x0 + 4));
                dd = dbit ? __ldg(reinterpret_cast<const uint4*>(dbit + x0)) : make_uint4(0, 0, 0, 0);
            } else {
                uint32_t r[8], d16[8];
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    r[k] = x0 + k < n ? perm[x0 + k] : 0xFFFFFFFFu;
                    d16[k] = (dbit && x0 + k < n) ? dbit[x0 + k] : CKS_NONE_INTERNAL;
                }
                r0 = make_uint4(r[0], r[1], r[2], r[3]);
                r1 = make_uint4(r[4], r[5], r[6], r[7]);
                dd = make_uint4(d16[0] | (d16[1] << 16), d16[2] | (d16[3] << 16), d16[4] | (d16[5] << 16),
                                d16[6] | (d16[7] << 16));
            }
            *reinterpret_cast<uint4*>(rid + x0) = r0;
            *reinterpret_cast<uint4*>(rid + x0 + 4) = r1;
            if (dbit) {
                if (edbit) *reinterpret_cast<uint4*>(edbit + x0) = dd;
                const uint32_t w[4] = {dd.x, dd.y, dd.z, dd.w};
#pragma unroll
                for (int k = 0; k < 4; k++) mn = min(mn, min(w[k] & 0xFFFF, w[k] >> 16));
            }
        }
        if (rmin) {
            for (uint32_t o = 1; o < tpn; o <<= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        if (g < groups && (g % tpn) == 0) {
            const uint64_t j = g / tpn;
            const uint64_t rem = n - j * fanout;
            node_cnt[j] = (uint32_t)(rem < fanout ? rem : fanout);
            if (rmin) rmin[j] = (uint16_t)mn;
        }
    }
}

static unsigned grid_warps(uint64_t nodes, int sms) {
    uint64_t want = (nodes + 7) / 8;                     // 8 warps per CTA
    if (want == 0) want = 1;
    uint64_t cap = (uint64_t)sms * 16;
    return (unsigned)(want < cap ? want : cap);
}

cudaError_t launch_bulk_leaves(const uint32_t* perm, const uint16_t* dbit, const BulkLevel& L,
                               uint32_t fanout, uint32_t per, uint32_t* node_cnt, uint32_t* rid,
                               uint16_t* edbit, uint16_t* rmin, int sms, cudaStream_t st) {
    const bool al = ((uintptr_t)perm % 16 == 0) && ((uintptr_t)rid % 16 == 0) &&
                    (!dbit || (uintptr_t)dbit % 16 == 0) && (!edbit || (uintptr_t)edbit % 16 == 0);
    if (per == fanout && fanout % 8 == 0 && fanout <= 256 && (fanout & (fanout - 1)) == 0 && al) {
        uint64_t groups = L.nodes * (fanout / 8);
        uint64_t want = (groups + 255) / 256;
        unsigned grid = (unsigned)(want < (uint64_t)sms * 16 ? want : (uint64_t)sms * 16);
        k_bulk_leaves_full<<<grid, 256, 0, st>>>(perm, dbit, L.entries, L.nodes, fanout, node_cnt, rid, edbit,
                                                 rmin);
        return cudaGetLastError();
    }
    k_bulk_leaves<<<grid_warps(L.nodes, sms), 256, 0, st>>>(perm, dbit, L, fanout, per, node_cnt, rid, edbit,
                                                            rmin);
    return cudaGetLastError();
}

cudaError_t launch_bulk_inner(const uint32_t* perm, const uint16_t* rmin_below, const BulkLevel& L,
                              uint64_t n, uint32_t fanout, uint32_t per, uint32_t* node_cnt,
                              uint32_t* rid, uint16_t* edbit, uint32_t* child, uint64_t inner_off,
                              uint16_t* rmin, int sms, cudaStream_t st, bool first_none) {
    k_bulk_inner<<<grid_warps(L.nodes, sms), 256, 0, st>>>(perm, rmin_below, L, n, fanout, per, node_cnt, rid,
                                                           edbit, child, inner_off, rmin, first_none ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace cks

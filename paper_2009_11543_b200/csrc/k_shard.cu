// k_shard.cu -- NEXT-4: the per-shard kernels of the sharded path that the
// single-GPU build does not have: the union of shard occupancies and the lower-bound rank
// of splitter keys in a locally sorted shard.
#include "cks_internal.h"

namespace cks {

// out[w] = OR over the nocc occupancies (u32[nocc][words]) -- NCCL has no OR reduction
__global__ void k_occ_union(const uint32_t* __restrict__ occ, uint32_t nocc, uint32_t words, uint32_t* __restrict__ out) {
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
        uint32_t v = 0;
        for (uint32_t g = 0; g < nocc; g++) v |= occ[(uint64_t)g * words + w];
        out[w] = v;
    }
}

// thread per query: binary search of (P, row id) in the sorted planes (plane np-1 most
// significant), row ids compared as rid_base + sorted_rid[i] against the query's
__global__ void k_rank_sorted(const uint32_t* __restrict__ planes, uint32_t np, uint64_t n,
                              const uint32_t* __restrict__ rid, uint64_t rid_base, const uint32_t* __restrict__ q,
                              uint32_t nq, unsigned long long* __restrict__ ranks) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nq) return;
    const uint32_t* qk = q + (uint64_t)t * (np + 1);
    const uint64_t qr = qk[np];
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        int c = 0;                                           // sign of element - query
        for (int w = (int)np - 1; w >= 0 && c == 0; w--) {
            const uint32_t a = planes[(uint64_t)w * n + mid], b = qk[w];
            c = a < b ? -1 : a > b ? 1 : 0;
        }
        if (c == 0) {
            const uint64_t a = rid_base + rid[mid];
            c = a < qr ? -1 : a > qr ? 1 : 0;
        }
        if (c < 0) lo = mid + 1;
        else hi = mid;
    }
    ranks[t] = lo;
}

cudaError_t launch_occ_union(const uint32_t* occ, uint32_t nocc, uint32_t words, uint32_t* out, cudaStream_t st) {
    k_occ_union<<<(words + 255) / 256 ? (words + 255) / 256 : 1, 256, 0, st>>>(occ, nocc, words, out);
    return cudaGetLastError();
}

cudaError_t launch_rank_sorted(const uint32_t* planes, uint32_t np, uint64_t n, const uint32_t* rid, uint64_t rid_base,
                               const uint32_t* q, uint32_t nq, unsigned long long* ranks, cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    k_rank_sorted<<<(nq + 127) / 128, 128, 0, st>>>(planes, np, n, rid, rid_base, q, nq, ranks);
    return cudaGetLastError();
}

}  // namespace cks

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

// part of every element: the number of splitters (in shared memory) <= (P_i, rid_base + i);
// per-part counts
__global__ void __launch_bounds__(256)
k_part_dest(const uint32_t* __restrict__ planes, uint32_t np, uint64_t n, uint64_t pitch,
            const uint32_t* __restrict__ spl, uint32_t nspl, uint64_t rid_base, uint32_t* __restrict__ dest,
            unsigned long long* __restrict__ counts) {
    extern __shared__ uint32_t s_sp[];                     // [nspl][np+1], then counts [nspl+1]
    uint32_t* s_cnt = s_sp + nspl * (np + 1);
    for (uint32_t i = threadIdx.x; i < nspl * (np + 1); i += blockDim.x) s_sp[i] = spl[i];
    for (uint32_t i = threadIdx.x; i <= nspl; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = nspl;                        // first splitter > element
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            const uint32_t* sk = s_sp + mid * (np + 1);
            int c = 0;                                     // sign of splitter - element
            for (int w = (int)np - 1; w >= 0 && c == 0; w--) {
                const uint32_t a = sk[w], b = planes[(uint64_t)w * pitch + i];
                c = a < b ? -1 : a > b ? 1 : 0;
            }
            if (c == 0) {
                const uint64_t a = sk[np], b = rid_base + i;
                c = a < b ? -1 : a > b ? 1 : 0;
            }
            if (c <= 0) lo = mid + 1;
            else hi = mid;
        }
        dest[i] = lo;
        atomicAdd(&s_cnt[lo], 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i <= nspl; i += blockDim.x)
        if (s_cnt[i]) atomicAdd(&counts[i], (unsigned long long)s_cnt[i]);
}

// right-aligned planes (cks_compress layout) -> left-aligned by `lead` bits (the refinement's
// P_M layout): out[q] = in[q] << lead | in[q-1] >> (32 - lead)
__global__ void k_align_left(const uint32_t* __restrict__ in, uint64_t in_pitch, uint32_t np, uint64_t n,
                             uint32_t lead, uint32_t* __restrict__ out, uint64_t out_pitch) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t lower = 0;
        for (uint32_t q = 0; q < np; q++) {
            const uint32_t v = in[(uint64_t)q * in_pitch + i];
            out[(uint64_t)q * out_pitch + i] = lead ? (v << lead) | (lower >> (32 - lead)) : v;
            lower = v;
        }
    }
}

__global__ void k_add_base(uint32_t* __restrict__ a, uint64_t n, uint32_t base) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] += base;
}

cudaError_t launch_part_dest(const uint32_t* planes, uint32_t np, uint64_t n, uint64_t pitch, const uint32_t* spl,
                             uint32_t nspl, uint64_t rid_base, uint32_t* dest, unsigned long long* counts, int sms,
                             cudaStream_t st) {
    cudaMemsetAsync(counts, 0, (size_t)(nspl + 1) * 8, st);
    if (n == 0) return cudaGetLastError();
    const size_t smem = ((size_t)nspl * (np + 1) + nspl + 1) * 4;
    uint64_t g = (n + 255) / 256;
    if (g > (uint64_t)sms * 8) g = (uint64_t)sms * 8;
    k_part_dest<<<(unsigned)g, 256, smem, st>>>(planes, np, n, pitch, spl, nspl, rid_base, dest, counts);
    return cudaGetLastError();
}

cudaError_t launch_align_left(const uint32_t* in, uint64_t in_pitch, uint32_t np, uint64_t n, uint32_t lead,
                              uint32_t* out, uint64_t out_pitch, int sms, cudaStream_t st) {
    if (n == 0 || np == 0) return cudaSuccess;
    uint64_t g = (n + 255) / 256;
    if (g > (uint64_t)sms * 8) g = (uint64_t)sms * 8;
    k_align_left<<<(unsigned)g, 256, 0, st>>>(in, in_pitch, np, n, lead, out, out_pitch);
    return cudaGetLastError();
}

cudaError_t launch_add_base(uint32_t* a, uint64_t n, uint32_t base, int sms, cudaStream_t st) {
    if (n == 0 || base == 0) return cudaSuccess;
    uint64_t g = (n + 255) / 256;
    if (g > (uint64_t)sms * 8) g = (uint64_t)sms * 8;
    k_add_base<<<(unsigned)g, 256, 0, st>>>(a, n, base);
    return cudaGetLastError();
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

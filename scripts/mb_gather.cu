// Microbenchmark: random 64-byte row gathers (the a7 row-order P_D compress on cfg4 reads
// 30 M random 64-byte key rows). Variants: each thread loads its own row with 4 x 16-byte
// loads (as k_compress_fixed) vs 4 lanes per row (one 16-byte load each), under the L2 fetch
// granularity limits 32/64/128. Prints ms per gather; run under ncu for DRAM bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_gather scripts/mb_gather.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void g_thread(const uint4* __restrict__ rows, const uint32_t* __restrict__ perm, uint64_t n,
                         uint32_t* __restrict__ out) {
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += T) {
        const uint4* p = rows + (uint64_t)__ldg(perm + i) * 4;
        uint4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2), d = __ldg(p + 3);
        out[i] = a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
    }
}

__global__ void g_quad(const uint4* __restrict__ rows, const uint32_t* __restrict__ perm, uint64_t n,
                       uint32_t* __restrict__ out) {
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x / 4;
    const int q = threadIdx.x & 3;
    for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 4; i < n; i += T) {
        const uint4* p = rows + (uint64_t)__ldg(perm + i) * 4;
        uint4 a = __ldg(p + q);
        uint32_t x = a.x ^ a.y ^ a.z ^ a.w;
        x ^= __shfl_xor_sync(0xffffffffu, x, 1);
        x ^= __shfl_xor_sync(0xffffffffu, x, 2);
        if (q == 0) out[i] = x;
    }
}

__global__ void g_seq(const uint4* __restrict__ rows, uint64_t n, uint32_t* __restrict__ out) {
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += T) {
        const uint4* p = rows + i * 4;
        uint4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2), d = __ldg(p + 3);
        out[i] = a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
    }
}

int main() {
    const uint64_t n = 30000000;
    uint4* rows; uint32_t *perm, *out;
    cudaMalloc(&rows, n * 64); cudaMalloc(&perm, n * 4); cudaMalloc(&out, n * 4);
    cudaMemset(rows, 1, n * 64);
    std::vector<uint32_t> h(n);
    for (uint64_t i = 0; i < n; i++) h[i] = (uint32_t)i;
    uint64_t s = 88172645463325252ull;
    for (uint64_t i = n - 1; i > 0; i--) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        uint64_t j = s % (i + 1);
        uint32_t t = h[i]; h[i] = h[j]; h[j] = t;
    }
    cudaMemcpy(perm, h.data(), n * 4, cudaMemcpyHostToDevice);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    size_t g0; cudaDeviceGetLimit(&g0, cudaLimitMaxL2FetchGranularity);
    printf("default L2 fetch granularity %zu\n", g0);
    for (int gran : {0, 32, 64, 128}) {
        if (gran) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        size_t g; cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
        for (int v = 0; v < 3; v++) {
            for (int per : {4, 8, 16}) {
                float best = 1e9;
                for (int it = 0; it < 5; it++) {
                    cudaEventRecord(e0);
                    if (v == 0) g_thread<<<sms * per, 256>>>(rows, perm, n, out);
                    else if (v == 1) g_quad<<<sms * per, 256>>>(rows, perm, n, out);
                    else g_seq<<<sms * per, 256>>>(rows, n, out);
                    cudaEventRecord(e1); cudaEventSynchronize(e1);
                    float ms; cudaEventElapsedTime(&ms, e0, e1);
                    if (ms < best) best = ms;
                }
                printf("gran %3zu %-6s ctas/sm %2d  %.3f ms  %.2f TB/s (rows)\n", g, v == 0 ? "thread" : v == 1 ? "quad" : "seq",
                       per, best, n * 64.0 / best / 1e9);
            }
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

// Microbenchmark (dev tool): throughput of scattered 32-bit RED.ADD into an
// L2-resident array, as K2 pass A issues them (d_in[v] += 1 for 2^28 edges into
// 2^24 counters), with uniform and Kronecker-skewed targets, and of the same
// count of scattered 4-byte loads (pass B's keep-bit lookups) from a 2 MB array.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__global__ void red_kernel(const uint32_t* __restrict__ idx, int64_t m, uint32_t* __restrict__ cnt) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[__ldcs(idx + i)], 1u);
}
__global__ void gather_kernel(const uint32_t* __restrict__ idx, int64_t m, const uint32_t* __restrict__ bits,
                              uint32_t* __restrict__ out) {
    uint32_t acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = __ldcs(idx + i);
        acc += (bits[v >> 5] >> (v & 31)) & 1u;
    }
    if (acc == 0xffffffffu) out[0] = acc;
}
__global__ void stream_kernel(const uint32_t* __restrict__ idx, int64_t m, uint32_t* __restrict__ out) {
    uint32_t acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        acc += __ldcs(idx + i);
    if (acc == 0xffffffffu) out[0] = acc;
}

int main() {
    const int64_t m = int64_t{1} << 28, n = int64_t{1} << 24;
    std::vector<uint32_t> h(m);
    uint32_t *d_idx, *d_cnt, *d_out;
    cudaMalloc(&d_idx, m * 4);
    cudaMalloc(&d_cnt, n * 4);
    cudaMalloc(&d_out, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int mode = 0; mode < 2; ++mode) {
        std::mt19937_64 g(1);
        for (int64_t i = 0; i < m; ++i) {
            uint64_t r = g();
            if (mode == 0) h[i] = (uint32_t)(r % n);
            else {  // Kronecker-like column: 24 bits, each 1 with p ~ 0.24 (b + d), then a fixed scramble
                const uint64_t r2 = g(), r3 = g();
                uint32_t v = 0;
                for (int b = 0; b < 8; ++b) {
                    v |= (uint32_t)(((r >> (8 * b)) & 255) < 61) << b;
                    v |= (uint32_t)(((r2 >> (8 * b)) & 255) < 61) << (b + 8);
                    v |= (uint32_t)(((r3 >> (8 * b)) & 255) < 61) << (b + 16);
                }
                h[i] = (v * 2654435761u) & (uint32_t)(n - 1);
            }
        }
        cudaMemcpy(d_idx, h.data(), m * 4, cudaMemcpyHostToDevice);
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(d_cnt, 0, n * 4);
            cudaEventRecord(e0);
            red_kernel<<<sms * 8, 512>>>(d_idx, m, d_cnt);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms_red = 0; cudaEventElapsedTime(&ms_red, e0, e1);
            cudaEventRecord(e0);
            gather_kernel<<<sms * 8, 512>>>(d_idx, m, d_cnt, d_out);  // 2 MB region = first 2^19 words
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms_g = 0; cudaEventElapsedTime(&ms_g, e0, e1);
            cudaEventRecord(e0);
            stream_kernel<<<sms * 8, 512>>>(d_idx, m, d_out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms_s = 0; cudaEventElapsedTime(&ms_s, e0, e1);
            printf("%s: 2^28 RED into 2^24 counters %.3f ms (%.2e/s) | 2^28 bit gathers (2 MB) %.3f ms | index stream 1 GB %.3f ms\n",
                   mode ? "skewed" : "uniform", ms_red, m / (ms_red * 1e-3), ms_g, ms_s);
        }
    }
    return 0;
}

// Dev reference point only (not product code): CUB onesweep radix sort of
// 2^28 u64 keys with 48 significant bits (the K1 key shape) and of 2^28 keys
// sorted on 24 bits (the K3 transpose shape), to calibrate the hand-written
// sort engine. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a cub_ref.cu -o cub_ref
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>
__global__ void fill(uint64_t* k, size_t n, int bits) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t x = i * 0x9e3779b97f4a7c15ull; x ^= x >> 31; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 29;
    k[i] = x & ((1ull << bits) - 1);
  }
}
int main() {
  const size_t n = 1ull << 28;
  uint64_t *a, *b; cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8);
  size_t tmp = 0; void* t = nullptr;
  cub::DeviceRadixSort::SortKeys(t, tmp, a, b, (int)n, 0, 48);
  cudaMalloc(&t, tmp);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int cfg = 0; cfg < 3; ++cfg) {
    int lo = cfg == 0 ? 0 : 25, hi = cfg == 0 ? 48 : 49;
    if (cfg == 2) { lo = 0; hi = 32; }
    for (int r = 0; r < 3; ++r) {
      fill<<<1184, 256>>>(a, n, cfg == 0 ? 48 : (cfg == 1 ? 49 : 32));
      cudaEventRecord(e0);
      cub::DeviceRadixSort::SortKeys(t, tmp, a, b, (int)n, lo, hi);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (r == 2) printf("cub SortKeys u64 n=2^28 bits[%d,%d): %.3f ms (%.1f Gkeys/s)\n", lo, hi, ms, n / (ms * 1e-3) / 1e9);
    }
  }
  // pairs: 24-bit keys (u32) + u32 values (transpose shape)
  uint32_t *k0, *k1, *v0, *v1; cudaMalloc(&k0, n * 4); cudaMalloc(&k1, n * 4); cudaMalloc(&v0, n * 4); cudaMalloc(&v1, n * 4);
  size_t tmp2 = 0; void* t2 = nullptr;
  cub::DeviceRadixSort::SortPairs(t2, tmp2, k0, k1, v0, v1, (int)n, 0, 24);
  cudaMalloc(&t2, tmp2);
  for (int r = 0; r < 3; ++r) {
    fill<<<1184, 256>>>(a, n, 24);
    cudaMemcpy2D(k0, 4, a, 8, 4, n, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0);
    cub::DeviceRadixSort::SortPairs(t2, tmp2, k0, k1, v0, v1, (int)n, 0, 24);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (r == 2) printf("cub SortPairs u32/u32 n=2^28 24 bits: %.3f ms\n", ms);
  }
  return 0;
}

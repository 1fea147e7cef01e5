// Microbenchmark round 2 (late): can the TMA unit serve as a second gather path
// beside the LSU? Random 16-byte cp.async.bulk copies (global -> shared, completed
// on an mbarrier) alone, and mixed with plain LDG gathers issued by the same
// warps, over an L2-resident table. Not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)
__device__ __forceinline__ unsigned hsh(unsigned x){ x^=x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }
__device__ __forceinline__ uint32_t smem_addr(const void* p){ return (uint32_t)__cvta_generic_to_shared(p); }

// Each warp owns an mbarrier and 32*KB slots of 16 bytes. Per round every lane
// issues KB bulk copies (TMA) and KL plain gathers (LSU); the warp then waits
// for its copies and consumes both.
template<int KB, int KL> __global__ void __launch_bounds__(256) k_mix(const double* __restrict__ a, unsigned mask, int rounds, double* out){
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  double2* slots = reinterpret_cast<double2*>(smem + 128) + (size_t)warp * 32 * (KB ? KB : 1);
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(bars + warp)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  double acc = 0; unsigned seed = (blockIdx.x * nw + warp) * 32 + lane; unsigned phase = 0;
  for (int r = 0; r < rounds; ++r) {
    if (KB) {
      if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_addr(bars + warp)), "r"(32u * KB * 16u) : "memory");
      __syncwarp();
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        const unsigned j = hsh(seed * 977u + r * 31u + k) & mask & ~1u;   // 16-byte aligned pair
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
                     :: "r"(smem_addr(slots + k * 32 + lane)), "l"(a + j), "r"(smem_addr(bars + warp)) : "memory");
      }
    }
    double x[KL ? KL : 1];
#pragma unroll
    for (int k = 0; k < KL; ++k) x[k] = __ldg(a + (hsh(seed * 131u + r * 17u + k + 7777u) & mask));
    if (KB) {
      unsigned done = 0;
      do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                        : "=r"(done) : "r"(smem_addr(bars + warp)), "r"(phase) : "memory"); } while (!done);
      phase ^= 1;
#pragma unroll
      for (int k = 0; k < KB; ++k) acc += slots[k * 32 + lane].x;
      __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < KL; ++k) acc += x[k];
  }
  if (acc == 1.2345) out[0] = acc;
}

template<int KB, int KL> void run(const double* g, unsigned mask, double* dout, int SM, double clk, const char* tag){
  const int rounds = 2048, threads = 256, blocks = SM * 6;
  const size_t smem = 128 + (size_t)(threads / 32) * 32 * (KB ? KB : 1) * 16;
  CK(cudaFuncSetAttribute(k_mix<KB, KL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms = 0;
  for (int rep = 0; rep < 3; ++rep) { cudaEventRecord(a); k_mix<KB, KL><<<blocks, threads, smem>>>(g, mask, rounds, dout); cudaEventRecord(b); CK(cudaEventSynchronize(b)); }
  cudaEventElapsedTime(&ms, a, b);
  const double n = (double)blocks * threads * rounds;
  printf("%-34s %5u MB: bulk %.3f /clk/SM + ldg %.3f /clk/SM = %.3f  (%.3f ms)\n", tag, (unsigned)((8ull * (mask + 1ull)) >> 20),
         n * KB / (ms * 1e-3) / (SM * clk), n * KL / (ms * 1e-3) / (SM * clk), n * (KB + KL) / (ms * 1e-3) / (SM * clk), ms);
}

int main(){ cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0)); int SM = p.multiProcessorCount; double clk = p.clockRate * 1e3;
  double* dout; CK(cudaMalloc(&dout, 64)); size_t bytes = 1ull << 28; double* g; CK(cudaMalloc(&g, bytes)); CK(cudaMemset(g, 0, bytes));
  for (unsigned lg : {13u, 23u}) { const unsigned mask = (1u << lg) - 1;
    run<0, 4>(g, mask, dout, SM, clk, "ldg only (4 per round)");
    run<0, 8>(g, mask, dout, SM, clk, "ldg only (8 per round)");
    run<4, 0>(g, mask, dout, SM, clk, "bulk-16B only (4 per round)");
    run<8, 0>(g, mask, dout, SM, clk, "bulk-16B only (8 per round)");
    run<1, 4>(g, mask, dout, SM, clk, "bulk 1 + ldg 4");
    run<2, 6>(g, mask, dout, SM, clk, "bulk 2 + ldg 6");
    run<4, 4>(g, mask, dout, SM, clk, "bulk 4 + ldg 4"); }
  return 0; }

// Microbenchmarks round 2: ranking via SMEM atomics with return, gather variants,
// SMEM/DSMEM random gathers, bucketed scatter stores. Not product code.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)
__device__ __forceinline__ unsigned hsh(unsigned x){ x^=x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }

template<int NB> __global__ void k_rank(size_t nkeys, unsigned* out){ extern __shared__ unsigned h[]; for(int i=threadIdx.x;i<NB;i+=blockDim.x)h[i]=0; __syncthreads(); unsigned acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<nkeys;i+=(size_t)gridDim.x*blockDim.x){ unsigned d=hsh((unsigned)i)&(NB-1); acc+=atomicAdd(&h[d],1u);} if(acc==0x1234567)out[0]=acc; }
__global__ void k_hashonly(size_t nkeys, unsigned* out){ unsigned acc=0; for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<nkeys;i+=(size_t)gridDim.x*blockDim.x) acc+=hsh((unsigned)i); if(acc==0x1234567)out[0]=acc; }

template<int MODE> __global__ void k_gather(const double* __restrict__ a, unsigned mask, size_t nops, double* out){ double acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<nops;i+=(size_t)gridDim.x*blockDim.x){ unsigned j=hsh((unsigned)i)&mask; const double* p=a+j; double v;
    if(MODE==0) v=__ldg(p);
    else if(MODE==1) asm volatile("ld.global.cg.f64 %0,[%1];":"=d"(v):"l"(p));
    else if(MODE==2) asm volatile("ld.global.nc.L1::no_allocate.f64 %0,[%1];":"=d"(v):"l"(p));
    else { // pairs of lanes share a line: lane^1 gathers neighbour
      unsigned jj=__shfl_sync(0xffffffffu,j,threadIdx.x&~1u); v=__ldg(a+((jj&~1u)|(threadIdx.x&1))); }
    acc+=v;} if(acc==1.2345) out[0]=acc; }
__global__ void k_gather4(const float* __restrict__ a, unsigned mask, size_t nops, float* out){ float acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<nops;i+=(size_t)gridDim.x*blockDim.x){ acc+=__ldg(a+(hsh((unsigned)i)&mask)); } if(acc==1.2345f) out[0]=acc; }
// streaming read with embedded gather: stream idx array (u32) and gather a[idx]
__global__ void k_spmv_like(const unsigned* __restrict__ idx, const double* __restrict__ val, const double* __restrict__ a, size_t n, double* out){ double acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){ acc+=val[i]*__ldg(a+idx[i]); } if(acc==1.2345) out[0]=acc; }
__global__ void k_fillidx(unsigned* idx, size_t n, unsigned mask){ for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) idx[i]=hsh((unsigned)i*7u+1u)&mask; }
// SMEM random gather
__global__ void k_sgather(size_t nops, int nd, double* out){ extern __shared__ double s[]; for(int i=threadIdx.x;i<nd;i+=blockDim.x) s[i]=i; __syncthreads(); double acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<nops;i+=(size_t)gridDim.x*blockDim.x){ acc+=s[hsh((unsigned)i)%nd]; } if(acc==1.2345) out[0]=acc; }
// DSMEM random gather across a cluster
__global__ void __cluster_dims__(8,1,1) k_dsgather(size_t nops, int nd, double* out){ extern __shared__ double s[]; cg::cluster_group cl=cg::this_cluster(); for(int i=threadIdx.x;i<nd;i+=blockDim.x) s[i]=i; cl.sync(); double acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<nops;i+=(size_t)gridDim.x*blockDim.x){ unsigned h=hsh((unsigned)i); double* rs=cl.map_shared_rank(s,(h>>24)&7); acc+=rs[h%nd]; } cl.sync(); if(acc==1.2345) out[0]=acc; }
// bucketed scatter: each key goes to bucket d (NB buckets), position by global atomic cursor per warp-group; simulates MSD scatter w/o smem staging
__global__ void k_bscatter(uint64_t* dst, unsigned* cursor, unsigned nb, size_t n, size_t cap){ for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){ unsigned d=hsh((unsigned)i)%nb; unsigned p=atomicAdd(cursor+d,1u); dst[(size_t)d*cap+p]=i; } }
__global__ void k_rscatter(uint64_t* dst, size_t n, unsigned mask){ for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){ dst[hsh((unsigned)i)&mask]=i; } }

int main(){ cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0)); int SM=p.multiProcessorCount; double clk=p.clockRate*1e3; cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  unsigned* uo; CK(cudaMalloc(&uo,64)); double* dout; CK(cudaMalloc(&dout,64)); size_t nk=1ull<<30;
#define TIME(call) for(int r_=0;r_<2;r_++){cudaEventRecord(a); call; cudaEventRecord(b); CK(cudaEventSynchronize(b));} cudaEventElapsedTime(&ms,a,b);
  TIME((k_hashonly<<<SM*8,256>>>(nk,uo))) printf("hash only: %.2f keys/clk/SM\n", nk/(ms*1e-3)/(SM*clk));
  TIME((k_rank<256><<<SM*8,256,256*4>>>(nk,uo))) printf("smem atomic-rank 256 bins: %.2f keys/clk/SM\n", nk/(ms*1e-3)/(SM*clk));
  TIME((k_rank<4096><<<SM*8,256,4096*4>>>(nk,uo))) printf("smem atomic-rank 4096 bins: %.2f keys/clk/SM\n", nk/(ms*1e-3)/(SM*clk));
  CK(cudaFuncSetAttribute(k_rank<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768*4));
  TIME((k_rank<32768><<<SM*2,1024,32768*4>>>(nk,uo))) printf("smem atomic-rank 32768 bins (1 blk/SM x1024): %.2f keys/clk/SM\n", nk/(ms*1e-3)/(SM*clk));
  double* g; CK(cudaMalloc(&g,1ull<<30)); CK(cudaMemset(g,0,1ull<<30)); size_t nops=1ull<<28;
  for(unsigned lg: {20u,23u,24u,26u}){
    TIME((k_gather<0><<<SM*8,512>>>(g,(1u<<lg)-1,nops,dout))) printf("gather8 ldg       %4u MB: %.2f /clk/SM\n",(8u<<lg)>>20,nops/(ms*1e-3)/(SM*clk));
    TIME((k_gather<1><<<SM*8,512>>>(g,(1u<<lg)-1,nops,dout))) printf("gather8 ld.cg     %4u MB: %.2f /clk/SM\n",(8u<<lg)>>20,nops/(ms*1e-3)/(SM*clk));
    TIME((k_gather<2><<<SM*8,512>>>(g,(1u<<lg)-1,nops,dout))) printf("gather8 noalloc   %4u MB: %.2f /clk/SM\n",(8u<<lg)>>20,nops/(ms*1e-3)/(SM*clk));
    TIME((k_gather<3><<<SM*8,512>>>(g,(1u<<lg)-1,nops,dout))) printf("gather8 pair-line %4u MB: %.2f /clk/SM\n",(8u<<lg)>>20,nops/(ms*1e-3)/(SM*clk));
    TIME((k_gather4<<<SM*8,512>>>((float*)g,(2u<<lg)-1,nops,(float*)dout))) printf("gather4 ldg       %4u MB: %.2f /clk/SM\n",(8u<<lg)>>20,nops/(ms*1e-3)/(SM*clk)); }
  // spmv-like streaming + gather over 59 MB and 128 MB targets
  size_t ne=1ull<<28; unsigned* idx; double* val; CK(cudaMalloc(&idx,ne*4)); CK(cudaMalloc(&val,ne*8)); CK(cudaMemset(val,0,ne*8));
  for(unsigned lg: {22u,23u,24u}){ k_fillidx<<<SM*8,512>>>(idx,ne,(1u<<lg)-1); CK(cudaDeviceSynchronize());
    TIME((k_spmv_like<<<SM*8,512>>>(idx,val,g,ne,dout))) printf("spmv-like over %u MB r: %.3f ms for %zu nnz -> %.2f nnz/clk/SM, stream %.0f GB/s\n",(8u<<lg)>>20,ms,ne,ne/(ms*1e-3)/(SM*clk),ne*12/(ms*1e-3)/1e9); }
  for(int nd: {4096, 24576}){ CK(cudaFuncSetAttribute(k_sgather, cudaFuncAttributeMaxDynamicSharedMemorySize, nd*8));
    TIME((k_sgather<<<SM*(nd>8192?1:4),1024,nd*8>>>(nops,nd,dout))) printf("smem gather8 over %d doubles: %.2f /clk/SM\n",nd,nops/(ms*1e-3)/(SM*clk)); }
  { int nd=24576; CK(cudaFuncSetAttribute(k_dsgather, cudaFuncAttributeMaxDynamicSharedMemorySize, nd*8));
    TIME((k_dsgather<<<144,1024,nd*8>>>(nops,nd,dout))) printf("dsmem(8) gather8 over 8x%d doubles: %.2f /clk/SM\n",nd,nops/(ms*1e-3)/(SM*clk)); }
  uint64_t* dst; CK(cudaMalloc(&dst,4ull<<30)); unsigned* cur; CK(cudaMalloc(&cur,1<<20)); size_t ns=1ull<<28;
  for(unsigned nb: {256u,4096u,32768u}){ CK(cudaMemset(cur,0,1<<20)); size_t cap=(ns/nb)*2; 
    for(int r=0;r<2;r++){ CK(cudaMemset(cur,0,1<<20)); cudaEventRecord(a); k_bscatter<<<SM*8,512>>>(dst,cur,nb,ns,cap); cudaEventRecord(b); CK(cudaEventSynchronize(b)); } cudaEventElapsedTime(&ms,a,b);
    printf("bucket scatter 8B (atomic cursor) %u buckets: %.3f ms, %.2f keys/clk/SM, %.0f GB/s written\n",nb,ms,ns/(ms*1e-3)/(SM*clk),ns*8/(ms*1e-3)/1e9); }
  TIME((k_rscatter<<<SM*8,512>>>(dst,ns,(1u<<28)-1))) printf("random 8B scatter over 2GB: %.3f ms, %.2f /clk/SM\n",ms,ns/(ms*1e-3)/(SM*clk));
  return 0; }

// Microbenchmarks that ground the K1/K2/K3 design: HBM streaming, SMEM atomic
// ranking throughput, L2 atomics, random gathers. Not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)

__device__ __forceinline__ uint64_t mix(uint64_t z){ z=(z^(z>>30))*0xbf58476d1ce4e5b9ULL; z=(z^(z>>27))*0x94d049bb133111ebULL; return z^(z>>31);}

__global__ void k_read(const int4* __restrict__ a, size_t n, int* out){ int4 acc={0,0,0,0}; for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){int4 v=__ldg(a+i); acc.x^=v.x;acc.y^=v.y;acc.z^=v.z;acc.w^=v.w;} if((acc.x^acc.y^acc.z^acc.w)==0x12345) out[0]=1; }
__global__ void k_copy(const int4* __restrict__ a, int4* b, size_t n){ for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x) b[i]=a[i]; }
// SMEM atomic histogram of random bins: nbins (pow2) per block
template<int NB> __global__ void k_satom(size_t nkeys, unsigned* out){ __shared__ unsigned h[NB]; for(int i=threadIdx.x;i<NB;i+=blockDim.x)h[i]=0; __syncthreads();
  uint64_t s = blockIdx.x*0x9e3779b97f4a7c15ULL + threadIdx.x*0x632BE59BD9B4E019ULL;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<nkeys;i+=(size_t)gridDim.x*blockDim.x){ s+=0x9e3779b97f4a7c15ULL; unsigned d=(unsigned)mix(s)&(NB-1); atomicAdd(&h[d],1u);} __syncthreads();
  for(int i=threadIdx.x;i<NB;i+=blockDim.x) if(h[i]==0xffffffff) out[0]=1; }
// baseline: same RNG without atomics
__global__ void k_rngonly(size_t nkeys, unsigned* out){ uint64_t s = blockIdx.x*0x9e3779b97f4a7c15ULL + threadIdx.x*0x632BE59BD9B4E019ULL; unsigned acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<nkeys;i+=(size_t)gridDim.x*blockDim.x){ s+=0x9e3779b97f4a7c15ULL; acc+=(unsigned)mix(s);} if(acc==0x1234567) out[0]=acc; }
// warp match_any ranking with warp-private histograms (256 bins)
__global__ void k_match(size_t nkeys, unsigned* out){ __shared__ unsigned h[32][256]; for(int i=threadIdx.x;i<32*256;i+=blockDim.x)(&h[0][0])[i]=0; __syncthreads();
  int w=threadIdx.x>>5, l=threadIdx.x&31; uint64_t s = blockIdx.x*0x9e3779b97f4a7c15ULL + threadIdx.x*0x632BE59BD9B4E019ULL; unsigned acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<nkeys;i+=(size_t)gridDim.x*blockDim.x){ s+=0x9e3779b97f4a7c15ULL; unsigned d=(unsigned)mix(s)&255;
    unsigned peers=__match_any_sync(0xffffffffu,d); int leader=31-__clz(peers); unsigned rank=__popc(peers&((1u<<l)-1)); unsigned base=0;
    if(l==leader){ base=h[w][d]; h[w][d]=base+__popc(peers);} base=__shfl_sync(0xffffffffu,base,leader); acc+=base+rank; }
  if(acc==0x1234567) out[0]=acc; }
// global red to random addresses in an array of nelem u32
__global__ void k_gred(unsigned* a, unsigned mask, size_t nops){ uint64_t s = blockIdx.x*0x9e3779b97f4a7c15ULL + threadIdx.x*0x632BE59BD9B4E019ULL;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<nops;i+=(size_t)gridDim.x*blockDim.x){ s+=0x9e3779b97f4a7c15ULL; atomicAdd(a+((unsigned)mix(s)&mask),1u);} }
// random 8B gather from array of nelem doubles
__global__ void k_gather(const double* __restrict__ a, unsigned mask, size_t nops, double* out){ uint64_t s = blockIdx.x*0x9e3779b97f4a7c15ULL + threadIdx.x*0x632BE59BD9B4E019ULL; double acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<nops;i+=(size_t)gridDim.x*blockDim.x){ s+=0x9e3779b97f4a7c15ULL; acc+=__ldg(a+((unsigned)mix(s)&mask));} if(acc==1.2345) out[0]=acc; }

int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev)); int l2=0; CK(cudaDeviceGetAttribute(&l2,cudaDevAttrL2CacheSize,dev)); int pl2=0; CK(cudaDeviceGetAttribute(&pl2,cudaDevAttrMaxPersistingL2CacheSize,dev));
  printf("dev %s SMs %d L2 %d persistL2max %d smemOptin %zu clock %d\n",p.name,p.multiProcessorCount,l2,pl2,p.sharedMemPerBlockOptin,p.clockRate);
  int SM=p.multiProcessorCount; cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  size_t bytes=4ull<<30; int4 *x,*y; CK(cudaMalloc(&x,bytes)); CK(cudaMalloc(&y,bytes)); CK(cudaMemset(x,1,bytes)); CK(cudaMemset(y,0,bytes)); int* o; CK(cudaMalloc(&o,64));
  size_t n=bytes/16;
  for(int blk: {256,512}) for(int g: {SM*4, SM*8, SM*16}){ for(int r=0;r<2;r++){ cudaEventRecord(a); k_read<<<g,blk>>>(x,n,o); cudaEventRecord(b); cudaEventSynchronize(b);} cudaEventElapsedTime(&ms,a,b); printf("read  blk%d g%d: %.1f GB/s\n",blk,g,bytes/ms/1e6); }
  for(int g: {SM*4, SM*8}){ for(int r=0;r<2;r++){ cudaEventRecord(a); k_copy<<<g,512>>>(x,y,n); cudaEventRecord(b); cudaEventSynchronize(b);} cudaEventElapsedTime(&ms,a,b); printf("copy g%d: %.1f GB/s (r+w)\n",g,2*bytes/ms/1e6); }
  size_t nk=1ull<<30; unsigned* uo; CK(cudaMalloc(&uo,64));
  auto rate=[&](const char* name){ cudaEventElapsedTime(&ms,a,b); double kps=nk/(ms*1e-3); printf("%-28s %.1f Gkeys/s = %.2f keys/clk/SM (at %d MHz)\n",name,kps/1e9,kps/(SM*(p.clockRate*1e3)),p.clockRate/1000); };
  for(int r=0;r<2;r++){cudaEventRecord(a); k_rngonly<<<SM*8,256>>>(nk,uo); cudaEventRecord(b); cudaEventSynchronize(b);} rate("rng only");
  for(int r=0;r<2;r++){cudaEventRecord(a); k_satom<256><<<SM*8,256>>>(nk,uo); cudaEventRecord(b); cudaEventSynchronize(b);} rate("smem atomic 256 bins");
  for(int r=0;r<2;r++){cudaEventRecord(a); k_satom<4096><<<SM*8,256>>>(nk,uo); cudaEventRecord(b); cudaEventSynchronize(b);} rate("smem atomic 4096 bins");
  for(int r=0;r<2;r++){cudaEventRecord(a); k_satom<8192><<<SM*4,512>>>(nk,uo); cudaEventRecord(b); cudaEventSynchronize(b);} rate("smem atomic 8192 bins");
  for(int r=0;r<2;r++){cudaEventRecord(a); k_match<<<SM*2,1024>>>(nk,uo); cudaEventRecord(b); cudaEventSynchronize(b);} rate("match_any warp-priv 256");
  unsigned* ga; CK(cudaMalloc(&ga,1ull<<30)); CK(cudaMemset(ga,0,1ull<<30)); size_t nops=1ull<<28;
  for(unsigned lg: {16u,20u,24u,26u,28u}){ for(int r=0;r<2;r++){cudaEventRecord(a); k_gred<<<SM*8,512>>>(ga,(1u<<lg)-1,nops); cudaEventRecord(b); cudaEventSynchronize(b);} cudaEventElapsedTime(&ms,a,b); printf("global atomicAdd random over 2^%u u32 (%u MB): %.1f Gops/s\n",lg,(4u<<lg)>>20,nops/(ms*1e-3)/1e9); }
  double* gd=(double*)ga; double* dout; CK(cudaMalloc(&dout,64));
  for(unsigned lg: {20u,23u,24u,25u,26u,27u}){ for(int r=0;r<2;r++){cudaEventRecord(a); k_gather<<<SM*8,512>>>(gd,(1u<<lg)-1,nops,dout); cudaEventRecord(b); cudaEventSynchronize(b);} cudaEventElapsedTime(&ms,a,b); printf("random 8B gather over %u MB: %.1f Gops/s (%.0f GB/s useful)\n",(8u<<lg)>>20,nops/(ms*1e-3)/1e9,nops*8/(ms*1e-3)/1e9); }
  return 0; }

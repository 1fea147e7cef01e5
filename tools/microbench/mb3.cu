// Microbenchmark round 2 (late): random 8-byte gathers through the texture path
// (tex1Dfetch<int2> on a linear texture object) against plain LDG, over
// L1-, L2- and HBM-sized tables. Not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)
__device__ __forceinline__ unsigned hsh(unsigned x){ x^=x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }

// HOT: 1 of 4 gathers goes to a 64 KB head (the SpMV's hot rows), the rest anywhere
template<int MODE, int HOT> __global__ void k_gather(const double* __restrict__ a, cudaTextureObject_t tex, unsigned mask, size_t nops, double* out){ double acc=0;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<nops;i+=(size_t)gridDim.x*blockDim.x){ unsigned h=hsh((unsigned)i); unsigned j=h&mask;
    if(HOT && (h>>30)==0) j&=8191u;
    double v;
    if(MODE==0) v=__ldg(a+j);
    else { int2 t=tex1Dfetch<int2>(tex,(int)j); v=__hiloint2double(t.y,t.x); }
    acc+=v;} if(acc==1.2345) out[0]=acc; }

int main(){ cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0)); int SM=p.multiProcessorCount; double clk=p.clockRate*1e3; cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  double* dout; CK(cudaMalloc(&dout,64));
#define TIME(call) for(int r_=0;r_<3;r_++){cudaEventRecord(a); call; cudaEventRecord(b); CK(cudaEventSynchronize(b));} cudaEventElapsedTime(&ms,a,b);
  size_t bytes=1ull<<29; double* g; CK(cudaMalloc(&g,bytes)); CK(cudaMemset(g,0,bytes)); size_t nops=1ull<<28;
  cudaResourceDesc rd{}; rd.resType=cudaResourceTypeLinear; rd.res.linear.devPtr=g; rd.res.linear.desc=cudaCreateChannelDesc<int2>(); rd.res.linear.sizeInBytes=bytes;
  cudaTextureDesc td{}; td.readMode=cudaReadModeElementType; cudaTextureObject_t tex; CK(cudaCreateTextureObject(&tex,&rd,&td,nullptr));
  for(unsigned lg: {13u,20u,23u,24u,26u}){
    TIME((k_gather<0,0><<<SM*8,512>>>(g,tex,(1u<<lg)-1,nops,dout))) printf("gather8 ldg      %6u KB: %.2f /clk/SM\n",(8u<<lg)>>10,nops/(ms*1e-3)/(SM*clk));
    TIME((k_gather<1,0><<<SM*8,512>>>(g,tex,(1u<<lg)-1,nops,dout))) printf("gather8 tex      %6u KB: %.2f /clk/SM\n",(8u<<lg)>>10,nops/(ms*1e-3)/(SM*clk));
    TIME((k_gather<0,1><<<SM*8,512>>>(g,tex,(1u<<lg)-1,nops,dout))) printf("gather8 ldg hot  %6u KB: %.2f /clk/SM\n",(8u<<lg)>>10,nops/(ms*1e-3)/(SM*clk));
    TIME((k_gather<1,1><<<SM*8,512>>>(g,tex,(1u<<lg)-1,nops,dout))) printf("gather8 tex hot  %6u KB: %.2f /clk/SM\n",(8u<<lg)>>10,nops/(ms*1e-3)/(SM*clk)); }
  return 0; }

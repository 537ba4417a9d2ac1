// Calibration microbenchmarks for the group-by design (not product code).
// Measures: HBM stream read / copy, SMEM atomics (u32/u64 add, u64 min, f64 add),
// global RED/ATOM on an L2-resident table, random L2 loads.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__device__ __forceinline__ uint64_t mix(uint64_t x){x^=x>>33;x*=0xff51afd7ed558ccdULL;x^=x>>33;x*=0xc4ceb9fe1a85ec53ULL;x^=x>>33;return x;}

__global__ void k_read(const uint4* __restrict__ a, size_t n, unsigned long long* out){
  size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x; uint32_t acc=0;
  for(;i<n;i+=st){uint4 v=__ldcs(a+i); acc^=v.x^v.y^v.z^v.w;}
  if(acc==0x12345678) atomicAdd(out,1ULL);
}
__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n){
  size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x;
  for(;i<n;i+=st){b[i]=__ldcs(a+i);}
}
template<int MODE>
__global__ void k_smem_atom(int iters, int slots_log2, unsigned long long* out){
  extern __shared__ unsigned long long sm[];
  int nslots=1<<slots_log2;
  for(int i=threadIdx.x;i<nslots;i+=blockDim.x) sm[i]=0;
  __syncthreads();
  uint64_t s=mix(blockIdx.x*1024+threadIdx.x);
  for(int it=0;it<iters;it++){
    s=s*6364136223846793005ULL+1442695040888963407ULL;
    int idx=(int)(s>>40)&(nslots-1);
    if(MODE==0) atomicAdd(&sm[idx],1ULL);
    else if(MODE==1) atomicAdd((unsigned*)&sm[idx],(unsigned)it);
    else if(MODE==6) atomicMin((unsigned*)&sm[idx],(unsigned)(s>>33));
    else if(MODE==2) atomicMin(&sm[idx],(unsigned long long)(s>>20));
    else if(MODE==3) atomicAdd((double*)&sm[idx],1.0);
    else if(MODE==4) { sm[idx]+=1; }            // racy plain RMW (cost reference)
    else if(MODE==5) { atomicAdd(&sm[idx],1ULL); atomicAdd(&sm[(idx+1)&(nslots-1)],(unsigned long long)it); atomicMin(&sm[(idx+2)&(nslots-1)],(unsigned long long)it); atomicMax(&sm[(idx+3)&(nslots-1)],(unsigned long long)it);}
  }
  __syncthreads();
  if(threadIdx.x==0) atomicAdd(out, sm[0]);
}
template<int MODE>
__global__ void k_glob_atom(unsigned long long* tab, int iters, int slots_log2){
  int nslots=1<<slots_log2;
  uint64_t s=mix(blockIdx.x*1024+threadIdx.x);
  for(int it=0;it<iters;it++){
    s=s*6364136223846793005ULL+1442695040888963407ULL;
    int idx=(int)(s>>36)&(nslots-1);
    if(MODE==0) atomicAdd(&tab[idx],1ULL);                 // RED.ADD.64
    else if(MODE==1) atomicAdd((double*)&tab[idx],1.0);    // RED.ADD.F64
    else if(MODE==2) atomicMin(&tab[idx],(unsigned long long)it);
    else if(MODE==3) { unsigned long long r=atomicCAS(&tab[idx],0ULL,(unsigned long long)it+1); if(r==0xdead) tab[0]=1; }
    else if(MODE==4) { unsigned long long v=__ldcg(&tab[idx]); if(v==0xdeadbeef) tab[1]=v; } // random L2 load
  }
}
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("dev %s SMs %d L2 %d MB smemOptin %zu KB clock %d MHz memclk %d MHz bus %d\n",p.name,p.multiProcessorCount,p.l2CacheSize>>20,p.sharedMemPerBlockOptin>>10,p.clockRate/1000,p.memoryClockRate/1000,p.memoryBusWidth);
  int nsm=p.multiProcessorCount;
  size_t bytes=4ull<<30; size_t n=bytes/16;
  uint4 *a,*b; CK(cudaMalloc(&a,bytes)); CK(cudaMalloc(&b,bytes)); CK(cudaMemset(a,1,bytes)); CK(cudaMemset(b,0,bytes));
  unsigned long long* out; CK(cudaMalloc(&out,8));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for(int bpsm: {4,8,16}){
    for(int r=0;r<3;r++){ cudaEventRecord(e0); k_read<<<nsm*bpsm,256>>>(a,n,out); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1);
    printf("read  bpsm=%d: %.1f GB/s\n",bpsm,bytes/ms/1e6);
    for(int r=0;r<3;r++){ cudaEventRecord(e0); k_copy<<<nsm*bpsm,256>>>(a,b,n/2); cudaEventRecord(e1); cudaEventSynchronize(e1);} cudaEventElapsedTime(&ms,e0,e1);
    printf("copy  bpsm=%d: %.1f GB/s (r+w)\n",bpsm,bytes/ms/1e6);
  }
  CK(cudaGetLastError());
  // smem atomics
  int iters=4096; int slog=14; size_t sb=(8ull<<slog);
  auto run_s=[&](auto kern,const char* name){
    cudaFuncSetAttribute(kern,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)sb);
    for(int r=0;r<2;r++){cudaEventRecord(e0); kern<<<nsm*1,1024,sb>>>(iters,slog,out); cudaEventRecord(e1); cudaEventSynchronize(e1);}
    cudaEventElapsedTime(&ms,e0,e1); double ops=(double)nsm*1024*iters; printf("smem %-22s: %.1f Gop/s  (%.2f lane-ops/clk/SM)\n",name,ops/ms/1e6, ops/(ms*1e-3)/nsm/(p.clockRate*1e3));
  };
  run_s(k_smem_atom<0>,"atomicAdd u64");
  run_s(k_smem_atom<1>,"atomicAdd u32");
  run_s(k_smem_atom<2>,"atomicMin u64");
  run_s(k_smem_atom<3>,"atomicAdd f64");
  run_s(k_smem_atom<4>,"plain RMW u64");
  run_s(k_smem_atom<6>,"atomicMin u32");
  run_s(k_smem_atom<5>,"4x(add,add,min,max)");
  CK(cudaGetLastError());
  unsigned long long* tab; CK(cudaMalloc(&tab,8ull<<22)); CK(cudaMemset(tab,0,8ull<<22));
  auto run_g=[&](auto kern,const char* name,int slog2){
    for(int r=0;r<2;r++){cudaEventRecord(e0); kern<<<nsm*4,512>>>(tab,1024,slog2); cudaEventRecord(e1); cudaEventSynchronize(e1);}
    cudaEventElapsedTime(&ms,e0,e1); double ops=(double)nsm*4*512*1024; printf("glob %-22s slots=2^%d: %.1f Gop/s\n",name,slog2,ops/ms/1e6);
  };
  for(int sl: {17,20,22}){
    run_g(k_glob_atom<0>,"RED.ADD.64",sl);
    run_g(k_glob_atom<1>,"RED.ADD.F64",sl);
    run_g(k_glob_atom<2>,"RED.MIN.64",sl);
    run_g(k_glob_atom<3>,"ATOM.CAS.64",sl);
    run_g(k_glob_atom<4>,"LDG.cg random",sl);
  }
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}

// NVLink pull variants, both directions at once: LDG.128, LDG.256 (v8), TMA bulk (cp.async.bulk) via smem.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("ERR %s %s:%d\n",cudaGetErrorString(e),__FILE__,__LINE__); return 1;}}while(0)
template<int U>
__global__ void copy16(const int4* __restrict__ src, int4* __restrict__ dst, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x*U + threadIdx.x; size_t stride=(size_t)gridDim.x*blockDim.x*U;
  for(; i < n; i += stride){
    int4 v[U];
    #pragma unroll
    for(int u=0;u<U;u++){ size_t k=i+u*blockDim.x; if(k<n) v[u]=src[k]; }
    #pragma unroll
    for(int u=0;u<U;u++){ size_t k=i+u*blockDim.x; if(k<n) dst[k]=v[u]; }
  }
}
struct alignas(32) v8 { uint32_t x[8]; };
__device__ __forceinline__ v8 ld32(const v8* p){ v8 r; asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r.x[0]),"=r"(r.x[1]),"=r"(r.x[2]),"=r"(r.x[3]),"=r"(r.x[4]),"=r"(r.x[5]),"=r"(r.x[6]),"=r"(r.x[7]) : "l"(p)); return r; }
__device__ __forceinline__ void st32(v8* p, const v8& r){ asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(p), "r"(r.x[0]),"r"(r.x[1]),"r"(r.x[2]),"r"(r.x[3]),"r"(r.x[4]),"r"(r.x[5]),"r"(r.x[6]),"r"(r.x[7]) : "memory"); }
template<int U>
__global__ void copy32(const v8* __restrict__ src, v8* __restrict__ dst, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x*U + threadIdx.x; size_t stride=(size_t)gridDim.x*blockDim.x*U;
  for(; i < n; i += stride){
    v8 v[U];
    #pragma unroll
    for(int u=0;u<U;u++){ size_t k=i+u*blockDim.x; if(k<n) v[u]=ld32(src+k); }
    #pragma unroll
    for(int u=0;u<U;u++){ size_t k=i+u*blockDim.x; if(k<n) st32(dst+k, v[u]); }
  }
}
// TMA bulk: one elected thread per CTA streams CHUNK-byte pieces through S smem stages
template<int S, int CHUNK>
__global__ void copy_bulk(const char* __restrict__ src, char* __restrict__ dst, size_t bytes){
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t mbar[S];
  if (threadIdx.x != 0) return;
  for (int s=0;s<S;s++){ uint32_t a=(uint32_t)__cvta_generic_to_shared(&mbar[s]); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;"::"r"(a)); }
  asm volatile("fence.mbarrier_init.release.cluster;":::"memory");
  size_t nchunks = bytes / CHUNK;
  uint32_t phase[S] = {0};
  int k = 0;
  // prologue: fill stages
  size_t c = blockIdx.x;
  size_t inflight[S]; int nin=0;
  for (int s=0; s<S && c < nchunks; s++, c += gridDim.x){
    uint32_t sm=(uint32_t)__cvta_generic_to_shared(smem + s*CHUNK), mb=(uint32_t)__cvta_generic_to_shared(&mbar[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"::"r"(mb),"r"(CHUNK):"memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"::"r"(sm),"l"(src + c*CHUNK),"r"(CHUNK),"r"(mb):"memory");
    inflight[s]=c; nin++;
  }
  for (int it=0; nin>0; it++){
    int s = it % S;
    uint32_t mb=(uint32_t)__cvta_generic_to_shared(&mbar[s]);
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }"::"r"(mb),"r"(phase[s]):"memory");
    phase[s]^=1;
    uint32_t sm=(uint32_t)__cvta_generic_to_shared(smem + s*CHUNK);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"::"l"(dst + inflight[s]*CHUNK),"r"(sm),"r"(CHUNK):"memory");
    asm volatile("cp.async.bulk.commit_group;":::"memory");
    asm volatile("cp.async.bulk.wait_group.read 0;":::"memory");
    nin--;
    if (c < nchunks){
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"::"r"(mb),"r"(CHUNK):"memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"::"r"(sm),"l"(src + c*CHUNK),"r"(CHUNK),"r"(mb):"memory");
      inflight[s]=c; nin++; c += gridDim.x;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;":::"memory");
}
int main(){
  size_t bytes = 1ull<<30;
  char *a[2], *b[2];
  for (int d=0; d<2; d++){ CK(cudaSetDevice(d)); CK(cudaMalloc(&a[d],bytes)); CK(cudaMalloc(&b[d],bytes)); CK(cudaMemset(a[d],1,bytes)); CK(cudaDeviceEnablePeerAccess(1-d,0));
    CK(cudaFuncSetAttribute(copy_bulk<4,32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4*32768));
    CK(cudaFuncSetAttribute(copy_bulk<6,32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6*32768));
    CK(cudaFuncSetAttribute(copy_bulk<8,16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8*16384)); }
  cudaEvent_t e0[2], e1[2]; cudaStream_t st[2];
  for (int d=0; d<2; d++){ CK(cudaSetDevice(d)); cudaEventCreate(&e0[d]); cudaEventCreate(&e1[d]); cudaStreamCreate(&st[d]); }
  const char* names[] = {"ldg128 x8", "ldg256 x4", "ldg256 x8", "bulk 4x32K", "bulk 6x32K", "bulk 8x16K"};
  for (int v=0; v<6; v++) for (int both=0; both<2; both++) for (int blocks: {148, 296, 592}) {
    float ms[2]={0,0};
    for (int rep=0; rep<2; rep++) {
      for (int d=0; d<(both?2:1); d++){ CK(cudaSetDevice(d)); cudaEventRecord(e0[d], st[d]);
        const char* src = a[1-d]; char* dst = b[d];
        for (int r=0;r<5;r++) {
          if (v==0) copy16<8><<<blocks*2,256,0,st[d]>>>((const int4*)src,(int4*)dst,bytes/16);
          if (v==1) copy32<4><<<blocks*2,256,0,st[d]>>>((const v8*)src,(v8*)dst,bytes/32);
          if (v==2) copy32<8><<<blocks*2,256,0,st[d]>>>((const v8*)src,(v8*)dst,bytes/32);
          if (v==3) copy_bulk<4,32768><<<blocks,32,4*32768,st[d]>>>(src,dst,bytes);
          if (v==4) copy_bulk<6,32768><<<blocks,32,6*32768,st[d]>>>(src,dst,bytes);
          if (v==5) copy_bulk<8,16384><<<blocks,32,8*16384,st[d]>>>(src,dst,bytes);
        }
        CK(cudaGetLastError());
        cudaEventRecord(e1[d], st[d]); }
      for (int d=0; d<(both?2:1); d++){ CK(cudaSetDevice(d)); CK(cudaEventSynchronize(e1[d])); cudaEventElapsedTime(&ms[d], e0[d], e1[d]); }
    }
    printf("%-11s %s ctas %4d: GPU0 %.1f GB/s", names[v], both?"both":"1dir", v<3?blocks*2:blocks, 5*bytes/ms[0]/1e6);
    if (both) printf("  GPU1 %.1f GB/s", 5*bytes/ms[1]/1e6);
    printf("\n");
  }
  // verify bulk result
  CK(cudaSetDevice(0)); char h[4]; CK(cudaMemcpy(h, b[0]+bytes-4, 4, cudaMemcpyDeviceToHost)); printf("check %d %d\n", h[0], h[3]);
  return 0;
}

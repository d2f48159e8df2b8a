// NVLink probe: pull vs push, one direction vs both directions at once (2 GPUs, one process).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("ERR %s %s:%d\n",cudaGetErrorString(e),__FILE__,__LINE__); return 1;}}while(0)
template<int U>
__global__ void copy(const int4* __restrict__ src, int4* __restrict__ dst, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x*U + threadIdx.x; size_t stride=(size_t)gridDim.x*blockDim.x*U;
  for(; i < n; i += stride){
    int4 v[U];
    #pragma unroll
    for(int u=0;u<U;u++){ size_t k=i+u*blockDim.x; if(k<n) v[u]=src[k]; }
    #pragma unroll
    for(int u=0;u<U;u++){ size_t k=i+u*blockDim.x; if(k<n) dst[k]=v[u]; }
  }
}
int main(){
  size_t bytes = 1ull<<30, nv = bytes/16;
  int4 *a[2], *b[2];
  for (int d=0; d<2; d++){ CK(cudaSetDevice(d)); CK(cudaMalloc(&a[d],bytes)); CK(cudaMalloc(&b[d],bytes)); CK(cudaMemset(a[d],1,bytes)); CK(cudaDeviceEnablePeerAccess(1-d,0)); }
  cudaEvent_t e0[2], e1[2]; cudaStream_t st[2];
  for (int d=0; d<2; d++){ CK(cudaSetDevice(d)); cudaEventCreate(&e0[d]); cudaEventCreate(&e1[d]); cudaStreamCreate(&st[d]); }
  for (int mode=0; mode<4; mode++) for (int blocks: {296, 444, 592, 1184}) {
    // mode 0: pull 1-dir (GPU0 reads GPU1), 1: pull both, 2: push 1-dir (GPU0 writes GPU1), 3: push both
    bool both = mode==1 || mode==3, push = mode>=2;
    float ms[2]={0,0};
    for (int rep=0; rep<2; rep++) {
      for (int d=0; d<(both?2:1); d++){ CK(cudaSetDevice(d)); cudaEventRecord(e0[d], st[d]);
        const int4* src = push ? a[d] : a[1-d]; int4* dst = push ? b[1-d] : b[d];
        for (int r=0;r<5;r++) copy<8><<<blocks,256,0,st[d]>>>(src,dst,nv);
        cudaEventRecord(e1[d], st[d]); }
      for (int d=0; d<(both?2:1); d++){ CK(cudaSetDevice(d)); CK(cudaEventSynchronize(e1[d])); cudaEventElapsedTime(&ms[d], e0[d], e1[d]); }
    }
    printf("%s %s blocks %4d: GPU0 %.1f GB/s%s", push?"push":"pull", both?"both":"1dir", blocks, 5*bytes/ms[0]/1e6, both?"":"\n");
    if (both) printf("  GPU1 %.1f GB/s\n", 5*bytes/ms[1]/1e6);
  }
  return 0;
}

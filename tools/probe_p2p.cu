// Probe: peer-access matrix and pull-copy bandwidth over NVLink (LDG.128 from peer, STG local).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("ERR %s %s:%d\n",cudaGetErrorString(e),__FILE__,__LINE__); return 1;}}while(0)
__global__ void pull(const int4* __restrict__ src, int4* __restrict__ dst, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x*4 + threadIdx.x; size_t stride=(size_t)gridDim.x*blockDim.x*4;
  for(; i < n; i += stride){
    int4 v[4];
    #pragma unroll
    for(int u=0;u<4;u++){ size_t k=i+u*blockDim.x; if(k<n) v[u]=src[k]; }
    #pragma unroll
    for(int u=0;u<4;u++){ size_t k=i+u*blockDim.x; if(k<n) dst[k]=v[u]; }
  }
}
int main(){
  int n; CK(cudaGetDeviceCount(&n)); printf("devices %d\n", n);
  for(int i=0;i<n;i++){ cudaDeviceProp p; cudaGetDeviceProperties(&p,i); printf("dev %d %s sms %d cc %d.%d\n",i,p.name,p.multiProcessorCount,p.major,p.minor);}
  if(n<2) return 0;
  size_t bytes = 1ull<<30; size_t nv = bytes/16;
  int4 *a,*b,*c; CK(cudaSetDevice(1)); CK(cudaMalloc(&a,bytes)); CK(cudaMemset(a,1,bytes));
  CK(cudaSetDevice(0)); CK(cudaMalloc(&b,bytes)); CK(cudaMalloc(&c,bytes)); CK(cudaDeviceEnablePeerAccess(1,0));
  int can; cudaDeviceCanAccessPeer(&can,0,1); printf("canAccess 0->1 %d\n",can);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for(int blocks : {148, 296, 592, 1184}) for(int th: {256,512}) {
    pull<<<blocks,th>>>(a,b,nv); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); for(int r=0;r<5;r++) pull<<<blocks,th>>>(a,b,nv); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1); printf("peer pull blocks %d th %d: %.1f GB/s\n",blocks,th, 5*bytes/ms/1e6);
  }
  cudaEventRecord(e0); for(int r=0;r<5;r++) pull<<<1184,512>>>(b,c,nv); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms,e0,e1); printf("local copy: %.1f GB/s (r+w)\n", 2*5*bytes/ms/1e6);
  cudaEventRecord(e0); for(int r=0;r<5;r++) cudaMemcpyPeerAsync(b,0,a,1,bytes); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1); printf("memcpyPeer: %.1f GB/s\n", 5*bytes/ms/1e6);
  return 0;
}

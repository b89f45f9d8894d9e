// Microbenchmark: shared-memory atomic / load throughput on B200 (design input for
// the query-count and DOPH bin-min kernels). Not part of the product path.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t xs(uint32_t x){ x^=x<<13; x^=x>>17; x^=x<<5; return x; }

template<int MODE>
__global__ void k(uint32_t* out, int iters, int mask){
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i <= mask; i += blockDim.x) s[i] = 0xFFFFFFFFu;
  __syncthreads();
  uint32_t x = 0x9E3779B9u * (threadIdx.x + 1 + blockIdx.x * 977);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    x = xs(x);
    int a = x & mask;
    if (MODE == 0) acc += s[a];                         // LDS random
    else if (MODE == 1) acc += atomicAdd(&s[a], 1u);    // ATOMS.ADD random w/ return
    else if (MODE == 2) atomicAdd(&s[a], 1u);           // ATOMS.ADD no return
    else if (MODE == 3) acc += atomicCAS(&s[a], 0xFFFFFFFFu, x); // CAS
    else if (MODE == 4) { if (x < s[a]) atomicMin(&s[a], x); }   // read-then-min
    else if (MODE == 5) atomicMin(&s[a], x);
    else if (MODE == 6) { unsigned long long* s64=(unsigned long long*)s; acc += (uint32_t)atomicCAS(&s64[a>>1], 0ull, (unsigned long long)x); }
  }
  __syncthreads();
  if (acc == 0x12345678u) out[0] = s[threadIdx.x & mask];
  if (threadIdx.x == 0) out[1 + blockIdx.x] = s[0];
}

__global__ void stream_read(const uint4* __restrict__ p, size_t n, uint32_t* out){
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main(){
  cudaDeviceProp pr; cudaGetDeviceProperties(&pr, 0);
  printf("dev %s SMs %d smemPerBlockOptin %zu L2 %d clock %d\n", pr.name, pr.multiProcessorCount, pr.sharedMemPerBlockOptin, pr.l2CacheSize, pr.clockRate);
  uint32_t* out; cudaMalloc(&out, 1<<20);
  int sms = pr.multiProcessorCount;
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"LDS","ATOMS.ADD(ret)","RED.S.ADD","ATOMS.CAS","LDS+cond-min","ATOMS.MIN","ATOMS.CAS64"};
  for (int mask : {255, 8191}) for (int mode = 0; mode < 7; ++mode) for (int blocks_per_sm : {1, 4}) {
    int threads = 256, iters = 4096;
    size_t sm = (mask + 1) * 4;
    void (*fn)(uint32_t*,int,int);
    switch(mode){case 0: fn=k<0>;break;case 1: fn=k<1>;break;case 2: fn=k<2>;break;case 3: fn=k<3>;break;case 4: fn=k<4>;break;case 5: fn=k<5>;break;default: fn=k<6>;}
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    int grid = sms * blocks_per_sm;
    fn<<<grid, threads, sm>>>(out, iters, mask);
    cudaEventRecord(a);
    fn<<<grid, threads, sm>>>(out, iters, mask);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)grid * threads * iters;
    printf("%-16s mask=%5d bps=%d : %.3f ms  %.2f Gop/s  %.2f lane-op/clk/SM(@1.9GHz)\n", names[mode], mask, blocks_per_sm, ms, ops/ms/1e6, ops/(ms*1e-3)/sms/1.9e9);
  }
  size_t bytes = 4ull<<30; uint4* p; cudaMalloc(&p, bytes); cudaMemset(p, 1, bytes);
  for (int g : {sms*2, sms*4, sms*8}) {
    stream_read<<<g, 512>>>(p, bytes/16, out);
    cudaEventRecord(a); stream_read<<<g, 512>>>(p, bytes/16, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); printf("stream read grid=%d: %.1f GB/s\n", g, bytes/ms/1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}

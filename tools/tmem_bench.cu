// Microbenchmark: tcgen05.ld (32x32b.x32) latency and issue cost, and the
// latency of a cp.async.bulk.tensor store issue, one CTA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I.. tools/tmem_bench.cu -o tools/tmem_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2104_05755_b200/csrc/sm100.cuh"

using namespace tpp::sm100;

__global__ void __launch_bounds__(128, 1) bench(unsigned long long* out, int mode) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  uint32_t v[32];
  uint32_t acc = 0;
  // warm
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
  tmem_ld_wait();
  for (int i = 0; i < 32; ++i) acc += v[i];
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < 16; ++it) {
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (it & 3) * 32, v);
    tmem_ld_wait();
    acc += v[it & 31];
  }
  unsigned long long t1 = clock64();
  // 4 loads in flight, one wait
  uint32_t w0[32], w1[32], w2[32], w3[32];
  unsigned long long t2 = clock64();
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), w0);
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 32, w1);
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 64, w2);
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + 96, w3);
  tmem_ld_wait();
  unsigned long long t3 = clock64();
  for (int i = 0; i < 32; ++i) acc += w0[i] ^ w1[i] ^ w2[i] ^ w3[i];
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / 16;
    out[1] = t3 - t2;
    out[2] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  for (int r = 0; r < 3; ++r) {
    bench<<<1, 128>>>(d, 0);
    cudaDeviceSynchronize();
    unsigned long long h[3];
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("tcgen05.ld 32x32b.x32 + wait: %llu cycles each (serial); 4 in flight + 1 wait: %llu cycles  %s\n", h[0],
           h[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

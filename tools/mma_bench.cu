// Microbenchmark: tcgen05.mma (kind::f16, SS operands) issue-to-completion
// throughput per shape, one CTA per SM, operands resident in shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I.. tools/mma_bench.cu -o tools/mma_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2104_05755_b200/csrc/sm100.cuh"

using namespace tpp::sm100;

template <int M, int N>
__global__ void __launch_bounds__(128, 1) bench(int iters, int a_shift, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(M, N);
    const uint64_t ad = sw128_kmajor_desc(smem_u32(sm) + a_shift * 128);
    const uint64_t bd = sw128_kmajor_desc(smem_u32(sm + 32 * 1024));
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) umma_f16(tmem, ad + (i & 3) * 2, bd + (i & 3) * 2, idesc, i > 0);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}

template <int M, int N>
void run(const char* name, int a_shift, unsigned long long* d) {
  const int iters = 4096;
  cudaFuncSetAttribute(bench<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  bench<M, N><<<148, 128, 80 * 1024>>>(iters, a_shift, d);
  cudaDeviceSynchronize();
  bench<M, N><<<148, 128, 80 * 1024>>>(iters, a_shift, d);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double cyc = (double)h / iters;
  printf("%-28s M=%3d N=%3d: %6.1f cycles/MMA  %7.0f MAC/cycle/SM  (floor %d)  %s\n", name, M, N, cyc,
         (double)M * N * 16 / cyc, (M < 128 ? 128 : M) * N / 256, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  run<128, 64>("SS", 0, d);
  run<128, 128>("SS", 0, d);
  run<128, 256>("SS", 0, d);
  run<64, 128>("SS", 0, d);
  run<64, 256>("SS", 0, d);
  run<128, 64>("SS, A row-shifted by 3", 3, d);
  run<128, 256>("SS, A row-shifted by 3", 3, d);
  return 0;
}

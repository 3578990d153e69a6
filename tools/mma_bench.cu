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


// Issue-pattern variants at M=128, N=64 (the conv tile): groups of G MMAs
// followed by C commits (to barriers nobody waits on until the end);
// conv = 9 taps with row-shifted A windows over a 32 KB halo and B from 72 KB
// of resident weights; alt = alternate two TMEM accumulators per group.
__global__ void __launch_bounds__(128, 1) pattern(int groups, int G, int C, int conv, int alt, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[3];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 104 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, 64);
    const uint64_t a0 = sw128_kmajor_desc(smem_u32(sm));
    const uint64_t b0 = sw128_kmajor_desc(smem_u32(sm + 32 * 1024));
    const unsigned long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      const uint32_t d = tmem + (alt ? (g & 1) * 64 : 0);
      for (int i = 0; i < G; ++i) {
        uint64_t ad, bd;
        if (conv) {
          const int tap = (i >> 2) % 9, kk = i & 3;
          ad = a0 + (uint64_t)((((tap / 3) * 64 + tap % 3) * 128) >> 4) + 2 * kk;
          bd = b0 + (uint64_t)((tap * 8192) >> 4) + 2 * kk;
        } else {
          ad = a0 + (i & 3) * 2;
          bd = b0 + (i & 3) * 2;
        }
        umma_f16(d, ad, bd, idesc, i > 0);
      }
      for (int c = 0; c < C; ++c) umma_commit(&bar[c]);
    }
    umma_commit(&bar[2]);
    mbar_wait(&bar[2], 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}

static void run_pattern(const char* name, int G, int C, int conv, int alt, unsigned long long* d) {
  const int groups = 4096 / G;
  cudaFuncSetAttribute(pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  pattern<<<148, 128, 110 * 1024>>>(groups, G, C, conv, alt, d);
  cudaDeviceSynchronize();
  pattern<<<148, 128, 110 * 1024>>>(groups, G, C, conv, alt, d);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-44s G=%2d C=%d: %6.1f cycles/MMA  %s\n", name, G, C, (double)h / (groups * G),
         cudaGetErrorString(cudaGetLastError()));
}


// The conv tile exactly as the product issues it (compile-time 3x3 taps, warp-
// collective issue, uniform warp index): 36 MMAs per tile into alternating
// accumulators, commits per tile (COMMITS = 0/1/2).
template <int COMMITS>
__global__ void __launch_bounds__(128, 1) conv_tile(int tiles, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[3];
  __shared__ uint32_t slot;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  for (int i = threadIdx.x; i < 104 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { for (int i = 0; i < 3; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, slot, 0);
  if (warp == 1) {
    const uint32_t idesc = idesc_bf16_f32(128, 64);
    const uint64_t a0 = sw128_kmajor_desc(smem_u32(sm));
    const uint64_t b0 = sw128_kmajor_desc(smem_u32(sm + 32 * 1024));
    const unsigned long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (t & 1) * 64;
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        const uint64_t ad = a0 + (uint64_t)((((tap / 3) * 64 + tap % 3) * 128) >> 4);
        const uint64_t bd = b0 + (uint64_t)((tap * 8192) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_f16_warp(d, ad + 2 * kk, bd + 2 * kk, idesc, (tap > 0 || kk > 0) ? 1u : 0u);
      }
      if (COMMITS >= 1) umma_commit_warp(&bar[0]);
      if (COMMITS >= 2) umma_commit_warp(&bar[1]);
    }
    umma_commit_warp(&bar[2]);
    mbar_wait(&bar[2], 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 32) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}

template <int COMMITS>
static void run_conv_tile(unsigned long long* d) {
  const int tiles = 200;
  cudaFuncSetAttribute(conv_tile<COMMITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  conv_tile<COMMITS><<<148, 128, 110 * 1024>>>(tiles, d);
  cudaDeviceSynchronize();
  conv_tile<COMMITS><<<148, 128, 110 * 1024>>>(tiles, d);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("conv tile (templated, warp issue)  commits=%d: %6.1f cycles/MMA  %s\n", COMMITS, (double)h / (tiles * 36),
         cudaGetErrorString(cudaGetLastError()));
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
  run_pattern("plain operands, one commit per group", 36, 0, 0, 0, d);
  run_pattern("plain operands", 36, 2, 0, 0, d);
  run_pattern("plain operands", 4, 1, 0, 0, d);
  run_pattern("conv taps (shifted A, 9 B blocks)", 36, 0, 1, 0, d);
  run_pattern("conv taps", 36, 2, 1, 0, d);
  run_pattern("conv taps, alternating accumulators", 36, 2, 1, 1, d);
  run_pattern("conv taps, alternating accumulators", 36, 1, 1, 1, d);
  run_conv_tile<0>(d);
  run_conv_tile<1>(d);
  run_conv_tile<2>(d);
  return 0;
}

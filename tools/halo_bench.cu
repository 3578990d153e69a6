// TMA feed throughput of the conv input halo (cfg 4 shape: N=256, H=W=56,
// 64 channels, [N][H][W][64] bf16): 148 persistent CTAs each walk their tiles
// (2 output rows) through a STAGES-deep ring, re-arming a stage as soon as it
// lands (no consumer).  Variants of the box geometry:
//   0: one box {64 ch, 64 px, 4 rows} at w = -1 (OOB px -1, 56..62)  [product]
//   1: four boxes {64, 56 px, 1 row} at w = 0, to smem row offsets r*8 KB + 128
//   2: one box {64, 56 px, 4 rows} at w = 0 (dense, throughput only)
//   3: one box {64, 64 px, 2 rows} at w = -1 (half the rows: a row-ring feed)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2104_05755_b200/csrc tools/halo_bench.cu -o tools/halo_bench
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace tpp::sm100;

constexpr int STAGES = 4;
constexpr int STAGE = 32 * 1024;

__global__ void __launch_bounds__(128, 1) halo_kernel(const __grid_constant__ CUtensorMap m, int variant, int tiles) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * STAGE);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  prefetch_tmap(&m);
  const int bytes = variant == 0 ? 32768 : variant == 3 ? 16384 : 4 * 56 * 128;  // 4: as 2
  int issued = 0;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++issued) {
    const int s = issued % STAGES;
    if (issued >= STAGES) mbar_wait(&full[s], ((issued / STAGES) - 1) & 1);  // the stage's previous load landed
    const int n = variant == 4 ? (tile / 28) % 4 : tile / 28, pr = tile % 28;  // 4: an L2-resident 3.2 MB window
    uint8_t* dst = sm + s * STAGE;
    mbar_arrive_expect_tx(&full[s], bytes);
    if (variant == 0) tma_load_5d(dst, &m, &full[s], 0, -1, 2 * pr - 1, 0, n);
    else if (variant == 1)
      for (int r = 0; r < 4; ++r) tma_load_5d(dst + r * 8192 + 128, &m, &full[s], 0, 0, 2 * pr - 1 + r, 0, n);
    else if (variant == 2) tma_load_5d(dst, &m, &full[s], 0, 0, 2 * pr - 1, 0, n);
    else if (variant == 3) tma_load_5d(dst, &m, &full[s], 0, -1, 2 * pr, 0, n);
    else tma_load_5d(dst, &m, &full[s], 0, 0, 2 * pr - 1, 0, n);
  }
  // drain the last STAGES loads
  for (int k = issued - STAGES; k < issued; ++k)
    if (k >= 0) mbar_wait(&full[k % STAGES], (k / STAGES) & 1);
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

int main() {
  const int N = 256, H = 56, W = 56;
  const size_t bytes = (size_t)N * H * W * 128;
  void* x;
  cudaMalloc(&x, bytes);
  cudaMemset(x, 0, bytes);
  void* flush;
  cudaMalloc(&flush, 512 << 20);
  const int tiles = N * 28;
  cudaFuncSetAttribute(halo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * STAGE + 2048);
  const char* names[] = {"box 64px x 4 rows at w=-1 (product)", "4 boxes 56px x 1 row", "box 56px x 4 rows (dense)",
                         "box 64px x 2 rows at w=-1", "box 56px x 4 rows, L2-resident window"};
  for (int v = 0; v < 5; ++v) {
    CUtensorMap m;
    cuuint64_t gd[5] = {64, (cuuint64_t)W, (cuuint64_t)H, 1, (cuuint64_t)N};
    cuuint64_t gs[4] = {128, (cuuint64_t)W * 128, (cuuint64_t)H * W * 128, (cuuint64_t)H * W * 128};
    cuuint32_t bd[5] = {64, v == 1 || v == 2 || v == 4 ? 56u : 64u, v == 1 ? 1u : (v == 3 ? 2u : 4u), 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, x, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
      cudaMemsetAsync(flush, it, 512 << 20);
      cudaEventRecord(e0);
      halo_kernel<<<148, 128, STAGES * STAGE + 2048>>>(m, v, tiles);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double moved = v != 3 ? (double)tiles * 4 * 56 * 128 : (double)tiles * 2 * 56 * 128;
    printf("%-40s %7.2f us  %7.1f GB/s (L2->SM, valid bytes)  %s\n", names[v], best * 1e3, moved / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

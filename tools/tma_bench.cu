// Microbenchmark: TMA ingest rate per SM for the box shapes the BRGEMM uses.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_bench tools/tma_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#include "../paper_2104_05755_b200/csrc/sm100.cuh"

using namespace tpp::sm100;

struct P {
  int kblocks, stages, bytes, rows, nload, reps, variant;
  const CUtensorMap* gmap;
};

__device__ unsigned long long g_ts[6][64];
__global__ void __launch_bounds__(96, 1) tma_kernel(const __grid_constant__ CUtensorMap m, P p, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + p.stages * p.bytes);
  uint64_t* empty = full + p.stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
    if (p.variant == 1) prefetch_tmap(&m);
    if (p.variant == 2) prefetch_tmap(p.gmap);
  }
  const CUtensorMap* mp = p.variant == 2 ? p.gmap : &m;
  __syncthreads();
  unsigned long long t0 = clock64();
  const int total = p.kblocks * p.reps;
  const int nprod = p.variant == 4 ? 2 : 1;
  const int pid = threadIdx.x == 0 ? 0 : (threadIdx.x == 64 ? 1 : -1);
  if (pid >= 0 && pid < nprod) {
    int s = pid, j = pid; uint32_t ph = 0;
    const int tile = (blockIdx.x % 8) * 256;
    for (int it = pid; it < total; it += nprod) {
      mbar_wait(&empty[s], ph ^ 1);
      mbar_arrive_expect_tx(&full[s], p.bytes);
      for (int l = 0; l < p.nload; ++l)
        tma_load_5d(smem + s * p.bytes + l * p.rows * 128, mp, &full[s], 0, 0, tile + l * p.rows, j, 0);
      s += nprod; if (s >= p.stages) { s -= p.stages; ph ^= 1; }
      j += nprod; if (j >= p.kblocks) j -= p.kblocks;
    }
  } else if (threadIdx.x == 32) {
    int s = 0; uint32_t ph = 0;
    for (int it = 0; it < total; ++it) {
      mbar_wait(&full[s], ph);
      if (blockIdx.x == 0 && it < 64) g_ts[1][it] = clock64() - t0;
      mbar_arrive(&empty[s]);
      if (++s == p.stages) { s = 0; ph ^= 1; }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  size_t n = 16ull * 4096 * 64;
  void* buf; cudaMalloc(&buf, n * 2); cudaMemset(buf, 0, n * 2);
  unsigned long long* cyc; cudaMalloc(&cyc, 4096 * 8);
  for (int rows : {64, 128, 256}) for (int nload : {1, 2}) { if (rows * nload > 256) continue;
    if (rows * nload > 256) continue;
    CUtensorMap m;
    cuuint64_t gd[5] = {64, 1, 4096, 16, 1}; cuuint64_t gs[4] = {128, 128, 4096ull*128, 16ull*4096*128};
    cuuint32_t bd[5] = {64, 1, (cuuint32_t)rows, 1, 1}; cuuint32_t es[5] = {1,1,1,1,1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, buf, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode failed %d\n", r); return 1; }
    CUtensorMap* gm; cudaMalloc(&gm, sizeof(CUtensorMap)); cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
    for (int variant : {0, 4}) for (int stages : {4}) for (int grid : {1, 148}) {
      P p{16, stages, rows * nload * 128, rows, nload, 64, variant, gm};
      int smem = stages * p.bytes + 2048;
      if (smem > 220 * 1024) continue;
      cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      tma_kernel<<<grid, 96, smem>>>(m, p, cyc);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      tma_kernel<<<grid, 96, smem>>>(m, p, cyc);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      std::vector<unsigned long long> h(grid); cudaMemcpy(h.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
      double avg = 0; for (auto v : h) avg += v; avg /= grid;
      double bytes = (double)p.kblocks * p.reps * p.bytes;
      if (false) { unsigned long long ts[6][64]; cudaMemcpyFromSymbol(ts, g_ts, sizeof(ts));
        for (int i = 0; i < 6; ++i) printf("  it %2d before-wait %6llu after-wait %6llu after-expect %6llu issued %6llu landed %6llu\n", i, ts[2][i], ts[3][i], ts[4][i], ts[0][i], ts[1][i]); }
      printf("variant %d box rows %3d x %d loads/stage (%6d B) stages %d grid %3d: per-SM %.1f B/cycle, total %.2f TB/s (%s)\n",
             variant, rows, nload, p.bytes, stages, grid, bytes / avg, bytes * grid / (ms * 1e-3) / 1e12,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

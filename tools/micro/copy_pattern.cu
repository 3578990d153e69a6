// Micro-benchmark: HBM copy efficiency vs per-column contiguity for a
// column-major 8192 x 4096 BF16 matrix.  Each warp instruction moves 512 B as
// (512 / seg) column segments of `seg` bytes; warps walk rows first.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

template <int SEG>
__global__ void copy_k(const uint4* __restrict__ in, uint4* __restrict__ out, int rows_b, int cols, int iters) {
  // rows_b: bytes per column; chunk = 16 B per lane
  constexpr int LPC = SEG / 16;  // lanes per column segment
  constexpr int CPI = 32 / LPC;  // columns per instruction
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x / 32);
  const int64_t colgroups = cols / CPI, segs = rows_b / SEG;
  const int64_t units = colgroups * segs;
  for (int64_t u = warp; u < units; u += nwarps) {
    const int64_t cg = u / segs, sg = u - cg * segs;
    const int64_t col = cg * CPI + lane / LPC;
    const int64_t off = (col * rows_b + sg * SEG) / 16 + (lane % LPC);
    out[off] = in[off];
  }
}

template <int SEG>
float run(const uint4* in, uint4* out, int rows_b, int cols) {
  const int blocks = 148 * 8, threads = 256;
  for (int i = 0; i < 3; ++i) copy_k<SEG><<<blocks, threads>>>(in, out, rows_b, cols, 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 20; ++i) copy_k<SEG><<<blocks, threads>>>(in, out, rows_b, cols, 1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 20;
}

int main() {
  const int rows = 8192, cols = 4096 * 3;  // 3x: operands larger than L2
  const int rows_b = rows * 2;
  const size_t bytes = (size_t)rows_b * cols;
  uint4 *in, *out;
  cudaMalloc(&in, bytes);
  cudaMalloc(&out, bytes);
  cudaMemset(in, 1, bytes);
  float t;
  t = run<128>(in, out, rows_b, cols); printf("seg 128B: %.1f us  %.0f GB/s\n", t * 1e3, 2.0 * bytes / t / 1e6);
  t = run<256>(in, out, rows_b, cols); printf("seg 256B: %.1f us  %.0f GB/s\n", t * 1e3, 2.0 * bytes / t / 1e6);
  t = run<512>(in, out, rows_b, cols); printf("seg 512B: %.1f us  %.0f GB/s\n", t * 1e3, 2.0 * bytes / t / 1e6);
  return 0;
}

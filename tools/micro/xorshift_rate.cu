// Micro-benchmark: xorshift128 keep-bit draws per second on the SMs, by how
// the three shifts are issued (ALU shifts vs IMAD.SHL / IMAD.HI on the FMA
// pipe) and by chains per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) { return __umulhi(a, b); }

template <int MODE>
__device__ __forceinline__ uint32_t step(uint32_t& x, uint32_t& y, uint32_t& z, uint32_t& w) {
  uint32_t t;
  if (MODE == 0) {        // IMAD.SHL + 2x IMAD.HI
    t = x ^ (x * 2048u);
    w = (w ^ mulhi(w, 1u << 13)) ^ (t ^ mulhi(t, 1u << 24));
  } else if (MODE == 1) { // all ALU shifts
    t = x ^ (x << 11);
    w = (w ^ (w >> 19)) ^ (t ^ (t >> 8));
  } else if (MODE == 2) { // IMAD.SHL, ALU right shifts
    t = x ^ (x * 2048u);
    w = (w ^ (w >> 19)) ^ (t ^ (t >> 8));
  } else {                // ALU left shift, one IMAD.HI
    t = x ^ (x << 11);
    w = (w ^ (w >> 19)) ^ (t ^ mulhi(t, 1u << 24));
  }
  x = y; y = z; z = w;
  return w;
}

template <int MODE, int CH, int ACC>
__global__ void __launch_bounds__(256) k(uint32_t* out, int n, uint32_t nthr) {
  uint32_t x[CH], y[CH], z[CH], w[CH], l[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    x[c] = threadIdx.x * 7 + c + 1; y[c] = blockIdx.x + 3; z[c] = 0x1234 + c; w[c] = 0x9876; l[c] = 0;
  }
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int u = 0; u < 32; ++u) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const uint32_t v = step<MODE>(x[c], y[c], z[c], w[c]);
        if (ACC == 0)
          asm("{ .reg .u32 d; add.cc.u32 d, %1, %2; addc.u32 %0, %0, %0; }" : "+r"(l[c]) : "r"(v), "r"(nthr));
        else
          l[c] = l[c] * 2u + (v >= ~nthr + 1u ? 1u : 0u);
      }
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) r ^= l[c] ^ w[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE, int CH, int ACC>
void run(uint32_t* out, const char* name) {
  const int blocks = 148 * 8, threads = 256, n = 64;
  k<MODE, CH, ACC><<<blocks, threads>>>(out, n, 0x19999A00u);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE, CH, ACC><<<blocks, threads>>>(out, n, 0x19999A00u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double draws = (double)blocks * threads * n * 32 * CH;
  printf("%-34s %7.2f Gdraws/s  (%.2f ns per 33.5M draws: %.1f us)\n", name, draws / ms / 1e6, 0.0,
         33554432.0 / (draws / ms / 1e6) / 1e3 * 1e3);
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  run<0, 1, 0>(out, "imad-shl+2imad-hi carry  ch1");
  run<0, 4, 0>(out, "imad-shl+2imad-hi carry  ch4");
  run<1, 1, 0>(out, "alu shifts carry         ch1");
  run<1, 4, 0>(out, "alu shifts carry         ch4");
  run<2, 4, 0>(out, "imad-shl, alu shr carry  ch4");
  run<3, 4, 0>(out, "alu shl, 1 imad-hi carry ch4");
  run<1, 4, 1>(out, "alu shifts setp-acc      ch4");
  run<2, 4, 1>(out, "imad-shl, alu shr setp   ch4");
  run<0, 4, 1>(out, "imad-shl+2imad-hi setp   ch4");
  return 0;
}

// K9: QUANTIZE / DEQUANTIZE TPPs (ops.py:447-469): symmetric per-tensor INT8.
//
// QUANTIZE (FP32 -> INT8): scale = amax / 127 (amax = max |x| over the view,
// in double; 1.0 when amax is not > 0, which includes a NaN amax because
// np.max propagates NaN), or the caller's scale; q = clip(rint(x / scale),
// -127, 127) with x / scale a double division and rint ties-to-even; NaN -> 0
// (numpy's float64 -> int8 cast of NaN on the reference's x86 host).
//   pass 1: |x| max as an unsigned atomicMax on the FP32 bit pattern (|x| >= 0
//           so the bit order is the value order; any NaN has bits above +inf,
//           so it wins exactly like np.max's NaN propagation)
//   pass 2: every thread derives the scale from the amax word, quantizes, and
//           thread 0 publishes the scale (double) for the caller.
// DEQUANTIZE (INT8 -> FP32): float32(q) * float32(scale), one rounding.

#include "common.cuh"

namespace tpp {

namespace {

__device__ __forceinline__ double scale_from_amax(uint32_t amax_bits) {
  const double amax = (double)__uint_as_float(amax_bits);
  return amax > 0.0 ? amax / 127.0 : 1.0;  // NaN amax -> 1.0
}

__global__ void quant_amax_kernel(DView in, uint32_t* __restrict__ amax_bits) {
  const int rows = in.rows;
  const int64_t n = (int64_t)rows * in.cols;
  uint32_t m = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / rows), i = (int)(e - (int64_t)j * rows);
    const uint32_t b = __float_as_uint(load_elem<float>(in, i, j)) & 0x7FFFFFFFu;
    m = b > m ? b : m;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint32_t t = __shfl_xor_sync(0xffffffffu, m, o);
    m = t > m ? t : m;
  }
  __shared__ uint32_t wmax[32];
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? wmax[threadIdx.x] : 0u;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const uint32_t t = __shfl_xor_sync(0xffffffffu, m, o);
      m = t > m ? t : m;
    }
    if (threadIdx.x == 0) atomicMax(amax_bits, m);
  }
}

__global__ void quant_apply_kernel(DView in, const uint32_t* __restrict__ amax_bits, int has_scale, double scale_in,
                                   int8_t* __restrict__ out, int out_ld, double* __restrict__ scale_out) {
  const double scale = has_scale ? scale_in : scale_from_amax(*amax_bits);
  if (blockIdx.x == 0 && threadIdx.x == 0 && scale_out) *scale_out = scale;
  const int rows = in.rows;
  const int64_t n = (int64_t)rows * in.cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / rows), i = (int)(e - (int64_t)j * rows);
    const double x = (double)load_elem<float>(in, i, j);
    double r = rint(__ddiv_rn(x, scale));
    r = r < -127.0 ? -127.0 : (r > 127.0 ? 127.0 : r);  // NaN falls through both tests
    out[i + (int64_t)j * out_ld] = (r == r) ? (int8_t)(int)r : (int8_t)0;
  }
}

__global__ void dequant_kernel(DView in, float scale, float* __restrict__ out, int out_ld) {
  const int rows = in.rows;
  const int64_t n = (int64_t)rows * in.cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / rows), i = (int)(e - (int64_t)j * rows);
    out[i + (int64_t)j * out_ld] = __fmul_rn(load_elem<float>(in, i, j), scale);
  }
}

unsigned grid_of(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (unsigned)(b < 148 * 8 ? (b > 0 ? b : 1) : 148 * 8);
}

}  // namespace

int launch_quantize(const DView& in, int has_scale, double scale, int8_t* out, int out_ld, uint32_t* amax_ws,
                    double* scale_out, cudaStream_t s) {
  const int64_t n = (int64_t)in.rows * in.cols;
  if (!has_scale) {
    cudaError_t e = cudaMemsetAsync(amax_ws, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess) return cuda_status(e, "quantize workspace");
    quant_amax_kernel<<<grid_of(n), 256, 0, s>>>(in, amax_ws);
    TPP_CUDA_LAUNCH_CHECK("quant_amax_kernel");
  }
  quant_apply_kernel<<<grid_of(n), 256, 0, s>>>(in, amax_ws, has_scale, scale, out, out_ld, scale_out);
  TPP_CUDA_LAUNCH_CHECK("quant_apply_kernel");
  return TPP_OK;
}

int launch_dequantize(const DView& in, double scale, float* out, int out_ld, cudaStream_t s) {
  const int64_t n = (int64_t)in.rows * in.cols;
  dequant_kernel<<<grid_of(n), 256, 0, s>>>(in, (float)scale, out, out_ld);
  TPP_CUDA_LAUNCH_CHECK("dequant_kernel");
  return TPP_OK;
}

}  // namespace tpp

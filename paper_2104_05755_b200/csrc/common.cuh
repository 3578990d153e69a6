// Shared device/host helpers for the sm_100a TPP library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/tpp_b200.h"
#include "launch.h"

namespace tpp {

// ---------------------------------------------------------------------------
// error plumbing (thread-local message, status codes of tpp_b200.h)
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_status(cudaError_t e, const char* what);
// the instantiation / grid of the last tensor-core launch of this thread
// (tpp_last_config(): tests assert which kernel a dispatch really runs)
void set_last_config(const std::string& cfg);

#define TPP_REQUIRE(cond, status, msg) \
  do {                                 \
    if (!(cond)) return ::tpp::fail((status), (msg)); \
  } while (0)

#define TPP_CUDA_LAUNCH_CHECK(what)                                   \
  do {                                                                \
    cudaError_t _e = cudaGetLastError();                              \
    if (_e != cudaSuccess) return ::tpp::cuda_status(_e, (what));     \
  } while (0)

inline int elem_size(int dtype) {
  switch (dtype) {
    case TPP_FP64: return 8;
    case TPP_FP32: return 4;
    case TPP_INT32: return 4;
    case TPP_BF16: return 2;
    case TPP_INT16: return 2;
    case TPP_INT8: return 1;
    default: return 0;
  }
}

inline int num_sms() {
  static int cached = -1;
  if (cached < 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      n = 148;
    cached = n;
  }
  return cached;
}

// ---------------------------------------------------------------------------
// precision codecs, bit-exact to dtypes.py:76-97
// ---------------------------------------------------------------------------
__device__ __forceinline__ float bf16_to_f32(uint16_t b) {
  return __uint_as_float(((uint32_t)b) << 16);
}

// fp32 -> bf16 RNE; NaN truncated with the quiet bit forced when the
// surviving payload would be empty (dtypes.py:92-97).  CUDA's own
// __float2bfloat16_rn canonicalises NaNs, so this is hand-written.
// Written with selects only: a per-element branch costs ~20 cycles of
// branch resolution on sm_100, more than the arithmetic.
__device__ __forceinline__ uint16_t f32_to_bf16(float v) {
  const uint32_t u = __float_as_uint(v);
  const uint32_t t = u >> 16;
  const uint32_t nan_bits = (t & 0x7Fu) == 0 ? (t | 0x40u) : t;
  const uint32_t rne = (u + 0x7FFFu + (t & 1u)) >> 16;
  return (uint16_t)((u & 0x7FFFFFFFu) > 0x7F800000u ? nan_bits : rne);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  return (uint32_t)f32_to_bf16(lo) | ((uint32_t)f32_to_bf16(hi) << 16);
}

// hardware cvt.rn.bf16x2.f32: identical RNE (incl. overflow to inf and
// subnormals) for numbers; NaNs come out canonical (0x7FFF)
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// Same result as pack_bf16x2, faster: the hardware convert, with the
// reference's NaN rule selected in for NaNs (branch-free).
__device__ __forceinline__ uint32_t pack2_bf16_ref(float lo, float hi) {
  const uint32_t r = cvt_bf16x2(lo, hi);
  const uint32_t lo_nan = (r & 0xFFFF0000u) | f32_to_bf16(lo);
  const uint32_t hi_nan = (r & 0x0000FFFFu) | ((uint32_t)f32_to_bf16(hi) << 16);
  return lo != lo ? (hi != hi ? pack_bf16x2(lo, hi) : lo_nan) : (hi != hi ? hi_nan : r);
}

// N pairs x[2i], x[2i+1] -> out[i]: hardware converts plus ONE (rarely taken)
// branch for the reference NaN rule, for the unrolled epilogues.
template <int N>
__device__ __forceinline__ void pack_bf16_ref_n(const float* x, uint32_t* out) {
  bool nan = false;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    out[i] = cvt_bf16x2(x[2 * i], x[2 * i + 1]);
    nan |= (x[2 * i] != x[2 * i]) | (x[2 * i + 1] != x[2 * i + 1]);
  }
  if (nan) {
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = pack_bf16x2(x[2 * i], x[2 * i + 1]);
  }
}

// ---------------------------------------------------------------------------
// GELU minimax erf table (approx.py:144-171, 267-288).  The 64 float32
// coefficients are the reference's Chebyshev fit (approx.py:127-158),
// regenerated bit-exactly by paper_2104_05755_b200/approx.py and pinned to the
// reference by tests/test_approx_table.py.  Layout: [c0 x16][c1 x16][c2 x16][c3 x16].
// ---------------------------------------------------------------------------
static __constant__ uint32_t c_gelu_bits[64] = {
    // c0
    0xAEAE681Eu, 0xB32420E3u, 0xB46F21C7u, 0xB5A33EBBu, 0xB6EC7C8Au, 0xB81FC150u, 0xB9622CB9u, 0xBA9278BCu,
    0xBBBCF479u, 0xBCCD9E2Cu, 0xBDB26317u, 0xBE22BAD9u, 0x3DFBB689u, 0x3F4AED87u, 0x3F7EBF65u, 0x3F7FFFF8u,
    // c1
    0x3F4C422Au, 0x3F4C4256u, 0x3F4C42E1u, 0x3F4C44EDu, 0x3F4C4D7Fu, 0x3F4C6D80u, 0x3F4CF01Eu, 0x3F4EC1AAu,
    0x3F5574E5u, 0x3F69140Cu, 0x3F8B4406u, 0x3F9EB67Bu, 0x3F59D017u, 0x3E24E948u, 0x3B36E9A9u, 0x344B69B4u,
    // c2
    0xB6A1804Au, 0xB88874BFu, 0xB9465A21u, 0xBA07D688u, 0xBAC480AEu, 0xBB8564E3u, 0xBC3D4771u, 0xBCF81BD3u,
    0xBDA2FCF8u, 0xBE39AED6u, 0xBEB3FEF1u, 0xBEEAF5B3u, 0xBE8F26B0u, 0xBD2B726Cu, 0xBA0A87BFu, 0xB2E1008Du,
    // c3
    0xBE080BCEu, 0xBE078F86u, 0xBE06EC32u, 0xBE05BC21u, 0xBE033668u, 0xBDFD2347u, 0xBDE9E244u, 0xBDC800F8u,
    0xBD885686u, 0xBCAED7D1u, 0x3D087A0Cu, 0x3D7034A9u, 0x3CFE59D0u, 0x3B6E6265u, 0x380B4821u, 0x30A57235u,
};
// host-visible copy of the same bits (for tests / tpp_gelu_table)
static const uint32_t h_gelu_bits[64] = {
    0xAEAE681Eu, 0xB32420E3u, 0xB46F21C7u, 0xB5A33EBBu, 0xB6EC7C8Au, 0xB81FC150u, 0xB9622CB9u, 0xBA9278BCu,
    0xBBBCF479u, 0xBCCD9E2Cu, 0xBDB26317u, 0xBE22BAD9u, 0x3DFBB689u, 0x3F4AED87u, 0x3F7EBF65u, 0x3F7FFFF8u,
    0x3F4C422Au, 0x3F4C4256u, 0x3F4C42E1u, 0x3F4C44EDu, 0x3F4C4D7Fu, 0x3F4C6D80u, 0x3F4CF01Eu, 0x3F4EC1AAu,
    0x3F5574E5u, 0x3F69140Cu, 0x3F8B4406u, 0x3F9EB67Bu, 0x3F59D017u, 0x3E24E948u, 0x3B36E9A9u, 0x344B69B4u,
    0xB6A1804Au, 0xB88874BFu, 0xB9465A21u, 0xBA07D688u, 0xBAC480AEu, 0xBB8564E3u, 0xBC3D4771u, 0xBCF81BD3u,
    0xBDA2FCF8u, 0xBE39AED6u, 0xBEB3FEF1u, 0xBEEAF5B3u, 0xBE8F26B0u, 0xBD2B726Cu, 0xBA0A87BFu, 0xB2E1008Du,
    0xBE080BCEu, 0xBE078F86u, 0xBE06EC32u, 0xBE05BC21u, 0xBE033668u, 0xBDFD2347u, 0xBDE9E244u, 0xBDC800F8u,
    0xBD885686u, 0xBCAED7D1u, 0x3D087A0Cu, 0x3D7034A9u, 0x3CFE59D0u, 0x3B6E6265u, 0x380B4821u, 0x30A57235u,
};
// copy the table into shared memory (call from >= 64 threads' worth of work, then sync)
__device__ __forceinline__ void load_gelu_table(float* dst, int tid, int nthreads) {
  for (int i = tid; i < 64; i += nthreads) dst[i] = __uint_as_float(c_gelu_bits[i]);
}
constexpr int kGeluBase = 244;          // (127 + emin) << 1, emin = -5
constexpr float kGeluRangeMax = 8.0f;   // first |x| that saturates

// h = minimax erf(x/sqrt2) with sign; coefficient table pointer may be
// shared memory (epilogues) or the constant bank.
__device__ __forceinline__ float gelu_h(float x, const float* tab) {
  float ax = fabsf(x);
  int idx = (int)(__float_as_uint(ax) >> 22) - kGeluBase;
  idx = idx < 0 ? 0 : (idx > 15 ? 15 : idx);
  float c0 = tab[idx], c1 = tab[16 + idx], c2 = tab[32 + idx], c3 = tab[48 + idx];
  float p = __fadd_rn(__fmul_rn(__fadd_rn(__fmul_rn(__fadd_rn(__fmul_rn(c3, ax), c2), ax), c1), ax), c0);
  if (ax >= kGeluRangeMax) p = 1.0f;
  return copysignf(p, x);
}

// gelu = (0.5*x) * (1 + h)   (approx.py:276, left-to-right as numpy)
__device__ __forceinline__ float gelu_fwd(float x, const float* tab) {
  float h = gelu_h(x, tab);
  return __fmul_rn(__fmul_rn(0.5f, x), __fadd_rn(1.0f, h));
}

// d/dx gelu = 0.5*(1+h) + (0.5*x)*hp  (approx.py:279-288, 174-183)
__device__ __forceinline__ float gelu_grad(float x, const float* tab) {
  float ax = fabsf(x);
  int idx = (int)(__float_as_uint(ax) >> 22) - kGeluBase;
  idx = idx < 0 ? 0 : (idx > 15 ? 15 : idx);
  float c1 = tab[16 + idx], c2 = tab[32 + idx], c3 = tab[48 + idx];
  float hp = __fadd_rn(__fmul_rn(__fadd_rn(__fmul_rn(__fmul_rn(3.0f, c3), ax), __fmul_rn(2.0f, c2)), ax), c1);
  if (ax >= kGeluRangeMax) hp = 0.0f;
  float h = gelu_h(x, tab);
  return __fadd_rn(__fmul_rn(0.5f, __fadd_rn(1.0f, h)), __fmul_rn(__fmul_rn(0.5f, x), hp));
}

// ReLU = np.maximum(x, 0): NaN propagates (payload kept), -0 -> +0 (ops.py:364)
__device__ __forceinline__ float relu_f(float x) {
  return (x != x) ? x : (x > 0.0f ? x : 0.0f);
}

// exp_taylor, FP32 path (approx.py:190-218)
__device__ __forceinline__ float exp_taylor(float x) {
  const float log2e = __uint_as_float(0x3FB8AA3Bu);
  const float c1 = __uint_as_float(0x3F316F7Du);
  const float c2 = __uint_as_float(0x3E781EEEu);
  const float c3 = __uint_as_float(0x3D656460u);
  float r = __fmul_rn(x, log2e);
  float n = rintf(r);  // round half to even, like np.rint
  float y = __fsub_rn(r, n);
  float q = __fadd_rn(__fmul_rn(__fadd_rn(__fmul_rn(__fadd_rn(__fmul_rn(c3, y), c2), y), c1), y), 1.0f);
  float nc = (n != n) ? 0.0f : fminf(fmaxf(n, -126.0f), 127.0f);
  int ni = (int)nc;
  float pow2 = __int_as_float((ni + 127) << 23);
  float out = __fmul_rn(q, pow2);
  if (x > 88.0f) out = __int_as_float(0x7F800000);
  if (x < -87.0f) out = 0.0f;
  return out;
}

// exp_taylor restricted to x <= 0 or NaN (softmax: x = v - max): bitwise the
// same results -- the x > 88 overflow branch and the upper exponent clamp
// cannot fire, and a NaN x gives NaN through q either way -- in 3 fewer
// instructions
__device__ __forceinline__ float exp_taylor_nonpos(float x) {
  const float log2e = __uint_as_float(0x3FB8AA3Bu);
  const float c1 = __uint_as_float(0x3F316F7Du);
  const float c2 = __uint_as_float(0x3E781EEEu);
  const float c3 = __uint_as_float(0x3D656460u);
  float r = __fmul_rn(x, log2e);
  float n = rintf(r);
  float y = __fsub_rn(r, n);
  float q = __fadd_rn(__fmul_rn(__fadd_rn(__fmul_rn(__fadd_rn(__fmul_rn(c3, y), c2), y), c1), y), 1.0f);
  int ni = (int)fmaxf(n, -126.0f);
  float out = __fmul_rn(q, __int_as_float((ni + 127) << 23));
  if (x < -87.0f) out = 0.0f;
  return out;
}

// Logical element (i, j) of a column-major view with ROW/COL/SCALAR broadcast
// (tensor.py:207-217), widened exactly; stores narrow once (RNE for BF16).
template <typename T>
__device__ __forceinline__ T load_elem(const DView& v, int i, int j) {
  const int pi = (v.bcast == TPP_BCAST_ROW || v.bcast == TPP_BCAST_SCALAR) ? 0 : i;
  const int pj = (v.bcast == TPP_BCAST_COL || v.bcast == TPP_BCAST_SCALAR) ? 0 : j;
  const int64_t idx = pi + (int64_t)pj * v.ld;
  switch (v.dtype) {
    case TPP_FP32: return (T) reinterpret_cast<const float*>(v.p)[idx];
    case TPP_BF16: return (T)bf16_to_f32(reinterpret_cast<const uint16_t*>(v.p)[idx]);
    case TPP_FP64: return (T) reinterpret_cast<const double*>(v.p)[idx];
    case TPP_INT32: return (T) reinterpret_cast<const int32_t*>(v.p)[idx];
    case TPP_INT8: return (T) reinterpret_cast<const int8_t*>(v.p)[idx];
    default: return T(0);
  }
}

template <typename T>
__device__ __forceinline__ void store_elem(void* p, int dtype, int64_t idx, T v) {
  switch (dtype) {
    case TPP_FP32: reinterpret_cast<float*>(p)[idx] = (float)v; break;
    case TPP_BF16: reinterpret_cast<uint16_t*>(p)[idx] = f32_to_bf16((float)v); break;
    case TPP_FP64: reinterpret_cast<double*>(p)[idx] = (double)v; break;
    default: break;
  }
}

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

}  // namespace tpp

// K1: BRGEMM in the reference's exact per-element order (SIMT).
//
// contraction.py:371-432: for every C element
//     acc  = beta==0 ? 0 : beta==1 ? C : C*beta          (410-415)
//     for i in batch:  part = +0;  for k ascending: part = part + a*b   (417-423)
//                      acc  = acc + part                  (424)
// Products and sums are separately rounded (no FMA), so the result is
// bitwise identical to the numpy reference for every dtype it supports
// (FP64, FP32, BF16 -> FP32 with exact widening, INT8 -> INT32 wrapping).
//
// Mapping: one thread owns TN consecutive C columns of one row; threads of a
// warp walk consecutive rows, so A loads coalesce and B loads broadcast.  The
// TN accumulation chains are independent, which is the ILP this kernel has
// (the per-element chain itself is inherently serial — that is the order).

#include "common.cuh"

namespace tpp {

template <typename T> struct Arith;
template <> struct Arith<float> {
  static __device__ __forceinline__ float mul(float x, float y) { return __fmul_rn(x, y); }
  static __device__ __forceinline__ float add(float x, float y) { return __fadd_rn(x, y); }
  static __device__ __forceinline__ float beta(double b) { return (float)b; }
};
template <> struct Arith<double> {
  static __device__ __forceinline__ double mul(double x, double y) { return __dmul_rn(x, y); }
  static __device__ __forceinline__ double add(double x, double y) { return __dadd_rn(x, y); }
  static __device__ __forceinline__ double beta(double b) { return b; }
};
template <> struct Arith<int32_t> {  // numpy int32 arithmetic wraps
  static __device__ __forceinline__ int32_t mul(int32_t x, int32_t y) {
    return (int32_t)((uint32_t)x * (uint32_t)y);
  }
  static __device__ __forceinline__ int32_t add(int32_t x, int32_t y) {
    return (int32_t)((uint32_t)x + (uint32_t)y);
  }
  static __device__ __forceinline__ int32_t beta(double b) { return (int32_t)b; }
};

template <typename TIn, typename TAcc> struct Widen;
template <> struct Widen<float, float> {
  static __device__ __forceinline__ float w(float v) { return v; }
};
template <> struct Widen<double, double> {
  static __device__ __forceinline__ double w(double v) { return v; }
};
template <> struct Widen<uint16_t, float> {
  static __device__ __forceinline__ float w(uint16_t v) { return bf16_to_f32(v); }
};
template <> struct Widen<int8_t, int32_t> {
  static __device__ __forceinline__ int32_t w(int8_t v) { return (int32_t)v; }
};

template <typename TIn, typename TAcc, int TN>
__global__ void __launch_bounds__(128)
brgemm_ordered_kernel(OrderedParams p) {
  using A = Arith<TAcc>;
  const int ncg = (p.n + TN - 1) / TN;  // column groups
  const int64_t elems = (int64_t)p.m * ncg;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= elems) return;
  const int mi = (int)(e % p.m);
  const int n0 = (int)(e / p.m) * TN;

  for (int64_t inst = blockIdx.y; inst < p.instances; inst += gridDim.y) {
    TAcc* c = reinterpret_cast<TAcc*>(p.c) + inst * p.inst_c;
    TAcc acc[TN];
    const TAcc bt = A::beta(p.beta);
#pragma unroll
    for (int t = 0; t < TN; ++t) {
      const int ni = n0 + t;
      if (ni >= p.n) { acc[t] = TAcc(0); continue; }
      if (p.beta == 0.0) acc[t] = TAcc(0);
      else if (p.beta == 1.0) acc[t] = c[mi + (int64_t)ni * p.ldc];
      else acc[t] = A::mul(c[mi + (int64_t)ni * p.ldc], bt);
    }
    for (int64_t i = 0; i < p.count; ++i) {
      const TIn* ab;
      const TIn* bb;
      if (p.mode == 0) {
        ab = reinterpret_cast<const TIn*>(p.a) + inst * p.inst_a + i * p.stride_a;
        bb = reinterpret_cast<const TIn*>(p.b) + inst * p.inst_b + i * p.stride_b;
      } else if (p.mode == 1) {
        ab = reinterpret_cast<const TIn*>(p.a) + p.a_offs[i];
        bb = reinterpret_cast<const TIn*>(p.b) + p.b_offs[i];
      } else {
        ab = reinterpret_cast<const TIn*>(p.a_ptrs[i]);
        bb = reinterpret_cast<const TIn*>(p.b_ptrs[i]);
      }
      TAcc part[TN];
#pragma unroll
      for (int t = 0; t < TN; ++t) part[t] = TAcc(0);
      const TIn* bcol[TN];
#pragma unroll
      for (int t = 0; t < TN; ++t) {
        const int ni = min(n0 + t, p.n - 1);
        bcol[t] = bb + (int64_t)ni * p.ldb;
      }
#pragma unroll 4
      for (int kk = 0; kk < p.k; ++kk) {
        TAcc av;
        if (p.vnni) {
          av = Widen<TIn, TAcc>::w(ab[(int64_t)(kk / p.alpha) * p.m * p.alpha +
                                      (int64_t)mi * p.alpha + (kk % p.alpha)]);
        } else {
          av = Widen<TIn, TAcc>::w(ab[mi + (int64_t)kk * p.lda]);
        }
#pragma unroll
        for (int t = 0; t < TN; ++t)
          part[t] = A::add(part[t], A::mul(av, Widen<TIn, TAcc>::w(bcol[t][kk])));
      }
#pragma unroll
      for (int t = 0; t < TN; ++t) acc[t] = A::add(acc[t], part[t]);
    }
#pragma unroll
    for (int t = 0; t < TN; ++t) {
      const int ni = n0 + t;
      if (ni < p.n) c[mi + (int64_t)ni * p.ldc] = acc[t];
    }
  }
}

template <typename TIn, typename TAcc>
static int launch_t(const OrderedParams& p, cudaStream_t s) {
  constexpr int TN = 4;
  const int ncg = (p.n + TN - 1) / TN;
  const int64_t elems = (int64_t)p.m * ncg;
  const int threads = 128;
  dim3 grid((unsigned)((elems + threads - 1) / threads),
            (unsigned)(p.instances < 65535 ? p.instances : 65535));
  brgemm_ordered_kernel<TIn, TAcc, TN><<<grid, threads, 0, s>>>(p);
  TPP_CUDA_LAUNCH_CHECK("brgemm_ordered_kernel");
  return TPP_OK;
}

// zero-count batches only apply the beta rule (contraction.py:410-425)
int launch_brgemm_ordered(const OrderedParams& p, int in_dtype, cudaStream_t s) {
  if (p.m == 0 || p.n == 0 || p.instances == 0) return TPP_OK;
  switch (in_dtype) {
    case TPP_FP32: return launch_t<float, float>(p, s);
    case TPP_FP64: return launch_t<double, double>(p, s);
    case TPP_BF16: return launch_t<uint16_t, float>(p, s);
    case TPP_INT8: return launch_t<int8_t, int32_t>(p, s);
    default: return fail(TPP_E_TENSOR, "unsupported BRGEMM input dtype");
  }
}

}  // namespace tpp

// K5: elementwise unary / binary / ternary / convert / reduce TPPs.
//
// Same blueprint as the reference (ops.py:1-8): load logical elements (with
// ROW/COL/SCALAR broadcast, tensor.py:207-217, and exact BF16 widening),
// compute in the compute precision (FP32; FP64 when an FP64 tensor is
// involved), store once (RNE narrowing for BF16, dtypes.py:82-97).  Every
// arithmetic op is a separately rounded IEEE op, so results are bitwise the
// reference's.  Views are column-major: element (i, j) at i + j*ld, and
// consecutive threads walk i, so every access coalesces.

#include "common.cuh"

namespace tpp {

template <typename T> struct Ops;
template <> struct Ops<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float sqrt_(float a) { return __fsqrt_rn(a); }
};
template <> struct Ops<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double sqrt_(double a) { return __dsqrt_rn(a); }
};

// np.maximum / np.minimum: NaN in either operand propagates
template <typename T>
__device__ __forceinline__ T np_max(T a, T b) { return (a != a) ? a : ((b != b) ? b : (a >= b ? a : b)); }
template <typename T>
__device__ __forceinline__ T np_min(T a, T b) { return (a != a) ? a : ((b != b) ? b : (a <= b ? a : b)); }

// ---------------------------------------------------------------------------
// unary (ops.py:284-386)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void unary_kernel(int kind, DView in, DView aux, void* out, int out_dtype, int out_ld,
                             uint8_t* mask_out) {
  __shared__ float tab[64];
  load_gelu_table(tab, threadIdx.x, blockDim.x);
  __syncthreads();
  using O = Ops<T>;
  const int rows = in.rows, cols = in.cols;
  const int bpc = (rows + 7) / 8;  // mask bytes per column (tensor.py:238-239)
  // one thread = 8 consecutive rows of one column = one mask byte
  const int64_t groups = (int64_t)bpc * cols;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(g / bpc);
    const int i0 = (int)(g % bpc) * 8;
    uint32_t bits = 0;
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u;
      if (i >= rows) break;
      T x = load_elem<T>(in, i, j);
      T r;
      switch (kind) {
        case TPP_UN_IDENTITY: r = x; break;
        case TPP_UN_ZERO: r = T(0); break;
        case TPP_UN_SQUARE: r = O::mul(x, x); break;
        case TPP_UN_INC: r = O::add(x, T(1)); break;
        case TPP_UN_DEC: r = O::sub(x, T(1)); break;
        case TPP_UN_SQRT: r = O::sqrt_(x); break;
        case TPP_UN_RECIPROCAL: r = O::div(T(1), x); break;
        case TPP_UN_RSQRT: r = O::div(T(1), O::sqrt_(x)); break;
        case TPP_UN_EXP: r = (T)exp_taylor((float)x); break;
        case TPP_UN_RELU:
          bits |= (x > T(0) ? 1u : 0u) << u;
          r = (x != x) ? x : (x > T(0) ? x : T(0));
          break;
        case TPP_UN_RELU_INV: {
          const uint8_t mb = reinterpret_cast<const uint8_t*>(aux.p)[(int64_t)j * bpc + (i >> 3)];
          r = ((mb >> (i & 7)) & 1) ? x : T(0);
          break;
        }
        case TPP_UN_GELU: r = (T)gelu_fwd((float)x, tab); break;
        case TPP_UN_GELU_INV: {
          const float xf = (float)load_elem<T>(aux, i, j);
          r = O::mul(x, (T)gelu_grad(xf, tab));
          break;
        }
        default: r = x; break;
      }
      store_elem<T>(out, out_dtype, i + (int64_t)j * out_ld, r);
    }
    if (mask_out) mask_out[(int64_t)j * bpc + i0 / 8] = (uint8_t)bits;
  }
}

int launch_unary(int kind, const DView& in, const DView& aux, void* out, int out_dtype, int out_ld,
                 uint8_t* mask_out, bool f64, cudaStream_t s) {
  const int64_t groups = (int64_t)((in.rows + 7) / 8) * in.cols;
  if (groups == 0) return TPP_OK;
  if (!f64) {
    const int rc = fast_unary(kind, in, aux, out, out_dtype, out_ld, mask_out, s);
    if (rc == 0) return TPP_OK;
    if (rc == 2) return cuda_status(cudaGetLastError(), "unary_vec_kernel");
  }
  const int threads = 256;
  int64_t blocks = (groups + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (f64)
    unary_kernel<double><<<(unsigned)blocks, threads, 0, s>>>(kind, in, aux, out, out_dtype, out_ld, mask_out);
  else
    unary_kernel<float><<<(unsigned)blocks, threads, 0, s>>>(kind, in, aux, out, out_dtype, out_ld, mask_out);
  TPP_CUDA_LAUNCH_CHECK("unary_kernel");
  return TPP_OK;
}

// ---------------------------------------------------------------------------
// binary (ops.py:747-782) and ternary MULADD/NMULADD (ops.py:796-816)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void nary_kernel(int arity, int kind, DView a, DView b, DView c, void* out, int rows,
                            int cols, int out_dtype, int out_ld) {
  using O = Ops<T>;
  const int64_t total = (int64_t)rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % rows), j = (int)(e / rows);
    const T x = load_elem<T>(a, i, j);
    const T y = load_elem<T>(b, i, j);
    T r;
    if (arity == 2) {
      switch (kind) {
        case TPP_BIN_ADD: r = O::add(x, y); break;
        case TPP_BIN_SUB: r = O::sub(x, y); break;
        case TPP_BIN_MUL: r = O::mul(x, y); break;
        case TPP_BIN_DIV: r = O::div(x, y); break;
        case TPP_BIN_MAX: r = np_max(x, y); break;
        default: r = np_min(x, y); break;
      }
    } else {
      const T z = load_elem<T>(c, i, j);
      const T prod = O::mul(x, y);
      r = kind == TPP_TER_MULADD ? O::add(z, prod) : O::sub(z, prod);
    }
    store_elem<T>(out, out_dtype, i + (int64_t)j * out_ld, r);
  }
}

int launch_nary(int arity, int kind, const DView& a, const DView& b, const DView& c, void* out,
                int rows, int cols, int out_dtype, int out_ld, bool f64, cudaStream_t s) {
  const int64_t total = (int64_t)rows * cols;
  if (total == 0) return TPP_OK;
  if (!f64) {
    const int rc = fast_nary(arity, kind, a, b, c, out, rows, cols, out_dtype, out_ld, s);
    if (rc == 0) return TPP_OK;
    if (rc == 2) return cuda_status(cudaGetLastError(), "nary_vec_kernel");
  }
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (f64)
    nary_kernel<double><<<(unsigned)blocks, threads, 0, s>>>(arity, kind, a, b, c, out, rows, cols, out_dtype, out_ld);
  else
    nary_kernel<float><<<(unsigned)blocks, threads, 0, s>>>(arity, kind, a, b, c, out, rows, cols, out_dtype, out_ld);
  TPP_CUDA_LAUNCH_CHECK("nary_kernel");
  return TPP_OK;
}

// contiguous BF16 -> BF16 / FP32 fast path for convert is the generic one:
// convert = IDENTITY unary with an output dtype (tensor.py:328-355)

// ---------------------------------------------------------------------------
// reduce (ops.py:484-522): fixed ascending fold, FP32 (FP64 for FP64) acc
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T fold(int op, T acc, T v) {
  switch (op) {
    case 0: return Ops<T>::add(acc, v);
    case 1: return Ops<T>::mul(acc, v);
    case 2: return np_min(acc, v);
    default: return np_max(acc, v);
  }
}

template <typename T>
__global__ void reduce_lines_kernel(DView in, int axis, int op, int squared, T* tmp_or_out,
                                    int out_dtype, void* out, int out_ld, int write_final) {
  // axis 0 (ROWS): line = row i, walk j ascending; axis 1 (COLS): line = column j, walk i
  const int nlines = axis == 0 ? in.rows : in.cols;
  const int len = axis == 0 ? in.cols : in.rows;
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nlines; l += gridDim.x * blockDim.x) {
    T acc;
    int start = 0;
    if (op == 0) acc = T(0);
    else if (op == 1) acc = T(1);
    else {
      T v = axis == 0 ? load_elem<T>(in, l, 0) : load_elem<T>(in, 0, l);
      if (squared) v = Ops<T>::mul(v, v);
      acc = v;
      start = 1;
    }
    for (int t = start; t < len; ++t) {
      T v = axis == 0 ? load_elem<T>(in, l, t) : load_elem<T>(in, t, l);
      if (squared) v = Ops<T>::mul(v, v);
      acc = fold(op, acc, v);
    }
    if (write_final) {
      // ROWS -> out (rows x 1): index l ; COLS -> out (1 x cols): index l*ld
      const int64_t idx = axis == 0 ? (int64_t)l : (int64_t)l * out_ld;
      store_elem<T>(out, out_dtype, idx, acc);
    } else {
      tmp_or_out[l] = acc;
    }
  }
}

template <typename T>
__global__ void reduce_all_final(const T* per_col, int cols, int op, int out_dtype, void* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  T acc;
  int start = 0;
  if (op == 0) acc = T(0);
  else if (op == 1) acc = T(1);
  else { acc = per_col[0]; start = 1; }
  for (int j = start; j < cols; ++j) acc = fold(op, acc, per_col[j]);
  store_elem<T>(out, out_dtype, 0, acc);
}

int launch_reduce(const DView& in, int axis, int op, int squared, void* out, int out_dtype,
                  int out_ld, void* scratch, bool f64, cudaStream_t s) {
  const int threads = 128;
  if (axis == 2) {
    // ALL: per-column fold over rows, then fold the columns (ops.py:519-521)
    const int blocks = (in.cols + threads - 1) / threads;
    if (f64) {
      reduce_lines_kernel<double><<<blocks, threads, 0, s>>>(in, 1, op, squared, (double*)scratch, out_dtype, out, out_ld, 0);
      reduce_all_final<double><<<1, 32, 0, s>>>((const double*)scratch, in.cols, op, out_dtype, out);
    } else {
      reduce_lines_kernel<float><<<blocks, threads, 0, s>>>(in, 1, op, squared, (float*)scratch, out_dtype, out, out_ld, 0);
      reduce_all_final<float><<<1, 32, 0, s>>>((const float*)scratch, in.cols, op, out_dtype, out);
    }
  } else {
    const int nlines = axis == 0 ? in.rows : in.cols;
    const int blocks = (nlines + threads - 1) / threads;
    if (f64)
      reduce_lines_kernel<double><<<blocks, threads, 0, s>>>(in, axis, op, squared, nullptr, out_dtype, out, out_ld, 1);
    else
      reduce_lines_kernel<float><<<blocks, threads, 0, s>>>(in, axis, op, squared, nullptr, out_dtype, out, out_ld, 1);
  }
  TPP_CUDA_LAUNCH_CHECK("reduce kernels");
  return TPP_OK;
}

}  // namespace tpp

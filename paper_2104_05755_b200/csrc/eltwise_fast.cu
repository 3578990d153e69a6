// K5/K6 fast paths: the memory-bound TPPs on dense operands at HBM speed.
//
// The generic kernels in eltwise.cu / transform.cu handle every view the
// reference allows (arbitrary ld, ROW/COL/SCALAR broadcast, any alpha, FP64).
// The common dense cases — column-major views with ld == rows (and rows a
// multiple of 8), FP32 compute, 16-byte aligned buffers — go through these
// kernels instead: 16-byte vector loads and stores, 8 elements (= one ReLU
// mask byte) per thread-step, grids sized to the SM count.  The per-element
// arithmetic is the generic kernels' (same separately rounded FP32 ops, same
// NaN / signed-zero rules, same RNE narrowing), so results are bit-identical.
//
// Transforms: TRANSPOSE is a 32x32 smem-tiled transpose of 2/4/8-byte
// elements; VNNI (alpha 2, BF16) interleaves column pairs with 16-byte
// accesses; VNNI_TO_VNNIT (alpha 2 -> 2, BF16) is a tiled transpose of 8-byte
// 2x2 blocks with the in-block swap done by byte permutes.

#include "common.cuh"

namespace tpp {

namespace fast {

// --- 8-element vectors ------------------------------------------------------
template <typename T> struct Vec8;
template <> struct Vec8<uint16_t> {  // BF16 storage
  static __device__ __forceinline__ void load(const void* p, int64_t g, float (&x)[8]) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + g);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      x[2 * q] = __uint_as_float(w[q] << 16);
      x[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
    }
  }
  static __device__ __forceinline__ void store(void* p, int64_t g, const float (&x)[8]) {
    uint32_t o[4];
    pack_bf16_ref_n<4>(x, o);
    reinterpret_cast<uint4*>(p)[g] = make_uint4(o[0], o[1], o[2], o[3]);
  }
};
template <> struct Vec8<float> {
  static __device__ __forceinline__ void load(const void* p, int64_t g, float (&x)[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p) + 2 * g);
    const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 2 * g + 1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  }
  static __device__ __forceinline__ void store(void* p, int64_t g, const float (&x)[8]) {
    reinterpret_cast<float4*>(p)[2 * g] = make_float4(x[0], x[1], x[2], x[3]);
    reinterpret_cast<float4*>(p)[2 * g + 1] = make_float4(x[4], x[5], x[6], x[7]);
  }
};

__device__ __forceinline__ float np_maxf(float a, float b) { return (a != a) ? a : ((b != b) ? b : (a >= b ? a : b)); }
__device__ __forceinline__ float np_minf(float a, float b) { return (a != a) ? a : ((b != b) ? b : (a <= b ? a : b)); }

// unary: the generic unary_kernel's per-element rules (eltwise.cu), FP32
template <typename TI, typename TO>
__global__ void __launch_bounds__(256)
unary_vec_kernel(int kind, const void* __restrict__ in, const void* __restrict__ aux, void* __restrict__ out,
                 uint8_t* __restrict__ mask_out, int64_t groups) {
  __shared__ float tab[64];
  load_gelu_table(tab, threadIdx.x, blockDim.x);
  __syncthreads();
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    float x[8], r[8];
    Vec8<TI>::load(in, g, x);
    uint32_t bits = 0;
    switch (kind) {
      case TPP_UN_IDENTITY:
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = x[u];
        break;
      case TPP_UN_ZERO:
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = 0.0f;
        break;
      case TPP_UN_SQUARE:
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = __fmul_rn(x[u], x[u]);
        break;
      case TPP_UN_INC:
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = __fadd_rn(x[u], 1.0f);
        break;
      case TPP_UN_DEC:
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = __fsub_rn(x[u], 1.0f);
        break;
      case TPP_UN_SQRT:
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = __fsqrt_rn(x[u]);
        break;
      case TPP_UN_RECIPROCAL:
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = __fdiv_rn(1.0f, x[u]);
        break;
      case TPP_UN_RSQRT:
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = __fdiv_rn(1.0f, __fsqrt_rn(x[u]));
        break;
      case TPP_UN_EXP:
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = exp_taylor(x[u]);
        break;
      case TPP_UN_RELU:
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          bits |= (x[u] > 0.0f ? 1u : 0u) << u;
          r[u] = (x[u] != x[u]) ? x[u] : (x[u] > 0.0f ? x[u] : 0.0f);
        }
        break;
      case TPP_UN_RELU_INV: {
        const uint32_t mb = reinterpret_cast<const uint8_t*>(aux)[g];
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = ((mb >> u) & 1) ? x[u] : 0.0f;
        break;
      }
      case TPP_UN_GELU:
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = gelu_fwd(x[u], tab);
        break;
      case TPP_UN_GELU_INV: {
        float xa[8];
        Vec8<TI>::load(aux, g, xa);
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = __fmul_rn(x[u], gelu_grad(xa[u], tab));
        break;
      }
      default:
#pragma unroll
        for (int u = 0; u < 8; ++u) r[u] = x[u];
        break;
    }
    Vec8<TO>::store(out, g, r);
    if (mask_out) mask_out[g] = (uint8_t)bits;
  }
}

// binary / ternary: the generic nary_kernel's rules, FP32
template <typename TI, typename TO>
__global__ void __launch_bounds__(256)
nary_vec_kernel(int arity, int kind, const void* __restrict__ a, const void* __restrict__ b,
                const void* __restrict__ c, void* __restrict__ out, int64_t groups) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    float x[8], y[8], r[8];
    Vec8<TI>::load(a, g, x);
    Vec8<TI>::load(b, g, y);
    if (arity == 2) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        switch (kind) {
          case TPP_BIN_ADD: r[u] = __fadd_rn(x[u], y[u]); break;
          case TPP_BIN_SUB: r[u] = __fsub_rn(x[u], y[u]); break;
          case TPP_BIN_MUL: r[u] = __fmul_rn(x[u], y[u]); break;
          case TPP_BIN_DIV: r[u] = __fdiv_rn(x[u], y[u]); break;
          case TPP_BIN_MAX: r[u] = np_maxf(x[u], y[u]); break;
          default: r[u] = np_minf(x[u], y[u]); break;
        }
      }
    } else {
      float z[8];
      Vec8<TI>::load(c, g, z);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float prod = __fmul_rn(x[u], y[u]);
        r[u] = kind == TPP_TER_MULADD ? __fadd_rn(z[u], prod) : __fsub_rn(z[u], prod);
      }
    }
    Vec8<TO>::store(out, g, r);
  }
}

inline unsigned grid_for(int64_t groups) {
  int64_t blocks = (groups + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  return (unsigned)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

inline bool dense(const DView& v, int rows) {
  return v.p && v.bcast == TPP_BCAST_NONE && v.ld == rows && reinterpret_cast<uintptr_t>(v.p) % 16 == 0;
}

// --- transforms ---------------------------------------------------------------
// out(j, i) = in(i, j) for an R x C column-major input (in: i + j*in_ld,
// out: j + i*out_ld), 32x32 tiles through smem, SWAP22: 8-byte elements are
// 2x2 BF16 blocks [w0 | w1] whose halves are exchanged (VNNI -> VNNIT)
template <typename E, bool SWAP22>
__global__ void __launch_bounds__(256)
tile_transpose_kernel(const E* __restrict__ in, int64_t in_ld, E* __restrict__ out, int64_t out_ld, int R, int C) {
  __shared__ E tile[32][33];
  const int tiles_i = (R + 31) / 32;
  const int i0 = (blockIdx.x % tiles_i) * 32, j0 = (blockIdx.x / tiles_i) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
  for (int jj = ty; jj < 32; jj += 8) {
    const int i = i0 + tx, j = j0 + jj;
    if (i < R && j < C) tile[jj][tx] = in[i + (int64_t)j * in_ld];
  }
  __syncthreads();
#pragma unroll
  for (int ii = ty; ii < 32; ii += 8) {
    const int j = j0 + tx, i = i0 + ii;
    if (i < R && j < C) {
      E v = tile[tx][ii];
      if constexpr (SWAP22) {
        // in block (words w0 = (a, b), w1 = (c, d)) -> out (w0' = (a, c), w1' = (b, d))
        const uint32_t w0 = (uint32_t)v, w1 = (uint32_t)(v >> 32);
        const uint32_t o0 = __byte_perm(w0, w1, 0x5410), o1 = __byte_perm(w0, w1, 0x7632);
        v = (E)o0 | ((E)o1 << 32);
      }
      out[j + (int64_t)i * out_ld] = v;
    }
  }
}

// 16-bit transpose with 32-bit global accesses: 64x64 tiles, element pairs
// along the contiguous dimension on both sides (R, C, lds even)
__global__ void __launch_bounds__(256)
transpose16_kernel(const uint32_t* __restrict__ in, int64_t in_ld2, uint32_t* __restrict__ out, int64_t out_ld2,
                   int R, int C) {
  __shared__ uint16_t tile[64][65];  // [j][i]; odd pitch: column reads conflict-free
  const int tiles_i = (R + 63) / 64;
  const int i0 = (blockIdx.x % tiles_i) * 64, j0 = (blockIdx.x / tiles_i) * 64;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int jj = ty; jj < 64; jj += 8) {
    const int i = i0 + 2 * tx, j = j0 + jj;
    if (i < R && j < C) {
      const uint32_t w = in[(i >> 1) + (int64_t)j * in_ld2];
      tile[jj][2 * tx] = (uint16_t)w;
      tile[jj][2 * tx + 1] = (uint16_t)(w >> 16);
    }
  }
  __syncthreads();
#pragma unroll
  for (int ii = ty; ii < 64; ii += 8) {
    const int j = j0 + 2 * tx, i = i0 + ii;
    if (i < R && j < C)
      out[(j >> 1) + (int64_t)i * out_ld2] = (uint32_t)tile[2 * tx][ii] | ((uint32_t)tile[2 * tx + 1][ii] << 16);
  }
}

// A/B switch for the 32-bit-access transpose below (experiments)
static bool use_word_transpose() {
  static const bool v = getenv("TPP_TRANSPOSE32") != nullptr;
  return v;
}

// 16-bit transpose with 16-byte global accesses, full 64x64 tiles (R, C
// multiples of 64, 16-byte aligned columns).  Each thread loads 8 rows of a
// column pair (two 16-byte loads), pairs them into 8 output words (row r+k,
// columns j, j+1) in registers, stages the words in a [64][33] shared tile
// (2-way bank conflicts on the writes, none on the reads) and stores 16-byte
// chunks of output rows.
__global__ void __launch_bounds__(256)
transpose16_v16_kernel(const uint16_t* __restrict__ in, int64_t in_ld, uint16_t* __restrict__ out, int64_t out_ld,
                       int R) {
  __shared__ uint32_t tile[64][33];  // [i][j/2]
  const int tiles_i = R / 64;
  const int i0 = (blockIdx.x % tiles_i) * 64, j0 = (blockIdx.x / tiles_i) * 64;
  const int t = threadIdx.x;
  {
    const int jp = t >> 3, c = t & 7;  // column pair (32), 8-row chunk (8)
    const uint16_t* src = in + i0 + 8 * c + (int64_t)(j0 + 2 * jp) * in_ld;
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(src));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(src + in_ld));
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      tile[8 * c + 2 * q][jp] = __byte_perm(aw[q], bw[q], 0x5410);      // row 2q: (a lo, b lo)
      tile[8 * c + 2 * q + 1][jp] = __byte_perm(aw[q], bw[q], 0x7632);  // row 2q+1: (a hi, b hi)
    }
  }
  __syncthreads();
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    const int i = (t >> 3) + 32 * pass, q = t & 7;  // output row, 16-byte chunk
    const uint4 v = make_uint4(tile[i][4 * q], tile[i][4 * q + 1], tile[i][4 * q + 2], tile[i][4 * q + 3]);
    *reinterpret_cast<uint4*>(out + j0 + 8 * q + (int64_t)(i0 + i) * out_ld) = v;
  }
}

// VNNI alpha 2, 16-bit: out column g = interleave(in columns 2g, 2g+1), with a
// zero column past lcols; 8 rows of one column pair per thread-step
__global__ void __launch_bounds__(256)
vnni2_kernel(const uint16_t* __restrict__ in, int64_t in_ld, uint16_t* __restrict__ out, int64_t out_ld, int M,
             int lcols, int groups_out_cols) {
  const int mv = M / 8;
  const int64_t total = (int64_t)mv * groups_out_cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int g = (int)(e / mv), m0 = (int)(e % mv) * 8;
    const int c0 = 2 * g, c1 = 2 * g + 1;
    const uint4 lo = __ldg(reinterpret_cast<const uint4*>(in + m0 + (int64_t)c0 * in_ld));
    const uint4 hi = c1 < lcols ? __ldg(reinterpret_cast<const uint4*>(in + m0 + (int64_t)c1 * in_ld))
                                : make_uint4(0, 0, 0, 0);
    const uint32_t a[4] = {lo.x, lo.y, lo.z, lo.w}, b[4] = {hi.x, hi.y, hi.z, hi.w};
    uint32_t o[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      o[2 * q] = __byte_perm(a[q], b[q], 0x5410);      // (a.lo, b.lo)
      o[2 * q + 1] = __byte_perm(a[q], b[q], 0x7632);  // (a.hi, b.hi)
    }
    uint4* dst = reinterpret_cast<uint4*>(out + 2 * (int64_t)m0 + (int64_t)g * out_ld);
    dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
    dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
  }
}

// DROPOUT_INV (ops.py:378-382) on dense views: group g = mask byte g
template <typename TI, typename TO>
__global__ void __launch_bounds__(256)
dropout_inv_vec_kernel(const void* __restrict__ in, const uint8_t* __restrict__ mask, float scale,
                       void* __restrict__ out, int64_t groups) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    float x[8];
    Vec8<TI>::load(in, g, x);
    const uint32_t b = __ldg(mask + g);
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = ((b >> u) & 1u) ? __fmul_rn(x[u], scale) : 0.0f;
    Vec8<TO>::store(out, g, x);
  }
}

}  // namespace fast

// 0 = handled, 1 = not applicable (fall back to the generic kernel)
int fast_unary(int kind, const DView& in, const DView& aux, void* out, int out_dtype, int out_ld, uint8_t* mask_out,
               cudaStream_t s) {
  using namespace fast;
  const int rows = in.rows;
  if (rows % 8 || out_ld != rows || !dense(in, rows) || reinterpret_cast<uintptr_t>(out) % 16) return 1;
  if ((in.dtype != TPP_BF16 && in.dtype != TPP_FP32) || (out_dtype != TPP_BF16 && out_dtype != TPP_FP32)) return 1;
  if (kind == TPP_UN_GELU_INV && (!dense(aux, rows) || aux.dtype != in.dtype)) return 1;
  if (kind == TPP_UN_RELU_INV && !aux.p) return 1;
  const int64_t groups = (int64_t)rows / 8 * in.cols;
  if (groups == 0) return 0;
  const unsigned grid = grid_for(groups);
  if (in.dtype == TPP_BF16 && out_dtype == TPP_BF16)
    unary_vec_kernel<uint16_t, uint16_t><<<grid, 256, 0, s>>>(kind, in.p, aux.p, out, mask_out, groups);
  else if (in.dtype == TPP_BF16)
    unary_vec_kernel<uint16_t, float><<<grid, 256, 0, s>>>(kind, in.p, aux.p, out, mask_out, groups);
  else if (out_dtype == TPP_BF16)
    unary_vec_kernel<float, uint16_t><<<grid, 256, 0, s>>>(kind, in.p, aux.p, out, mask_out, groups);
  else
    unary_vec_kernel<float, float><<<grid, 256, 0, s>>>(kind, in.p, aux.p, out, mask_out, groups);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int fast_nary(int arity, int kind, const DView& a, const DView& b, const DView& c, void* out, int rows, int cols,
              int out_dtype, int out_ld, cudaStream_t s) {
  using namespace fast;
  if (rows % 8 || out_ld != rows || !dense(a, rows) || !dense(b, rows) || reinterpret_cast<uintptr_t>(out) % 16)
    return 1;
  if (arity == 3 && !dense(c, rows)) return 1;
  const int dt = a.dtype;
  if ((dt != TPP_BF16 && dt != TPP_FP32) || b.dtype != dt || (arity == 3 && c.dtype != dt)) return 1;
  if (out_dtype != TPP_BF16 && out_dtype != TPP_FP32) return 1;
  const int64_t groups = (int64_t)rows / 8 * cols;
  if (groups == 0) return 0;
  const unsigned grid = grid_for(groups);
  if (dt == TPP_BF16 && out_dtype == TPP_BF16)
    nary_vec_kernel<uint16_t, uint16_t><<<grid, 256, 0, s>>>(arity, kind, a.p, b.p, c.p, out, groups);
  else if (dt == TPP_BF16)
    nary_vec_kernel<uint16_t, float><<<grid, 256, 0, s>>>(arity, kind, a.p, b.p, c.p, out, groups);
  else if (out_dtype == TPP_BF16)
    nary_vec_kernel<float, uint16_t><<<grid, 256, 0, s>>>(arity, kind, a.p, b.p, c.p, out, groups);
  else
    nary_vec_kernel<float, float><<<grid, 256, 0, s>>>(arity, kind, a.p, b.p, c.p, out, groups);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

// kind: 0 TRANSPOSE, 1 VNNI, 2 VNNI_TO_VNNIT (launch_transform's numbering)
int fast_transform(int kind, int esize, const void* in, int in_ld, void* out, int out_rows, int out_cols,
                   int out_ld, int alpha, int alpha_out, int lrows, int lcols, cudaStream_t s) {
  using namespace fast;
  if (kind == 0) {
    // in is out_cols x out_rows (R x C), out is out_rows x out_cols
    const int R = out_cols, C = out_rows;
    const unsigned grid = (unsigned)(((R + 31) / 32) * ((C + 31) / 32));
    if (grid == 0) return 0;
    switch (esize) {
      case 2:
        if (R % 64 == 0 && C % 64 == 0 && in_ld % 8 == 0 && out_ld % 8 == 0 && reinterpret_cast<uintptr_t>(in) % 16 == 0 &&
            reinterpret_cast<uintptr_t>(out) % 16 == 0 && !use_word_transpose()) {
          const unsigned g64 = (unsigned)((R / 64) * (C / 64));
          fast::transpose16_v16_kernel<<<g64, 256, 0, s>>>((const uint16_t*)in, in_ld, (uint16_t*)out, out_ld, R);
        } else if (R % 2 == 0 && C % 2 == 0 && in_ld % 2 == 0 && out_ld % 2 == 0 && reinterpret_cast<uintptr_t>(in) % 4 == 0 &&
            reinterpret_cast<uintptr_t>(out) % 4 == 0) {
          const unsigned g64 = (unsigned)(((R + 63) / 64) * ((C + 63) / 64));
          fast::transpose16_kernel<<<g64, 256, 0, s>>>((const uint32_t*)in, in_ld / 2, (uint32_t*)out, out_ld / 2, R, C);
        } else {
          fast::tile_transpose_kernel<uint16_t, false><<<grid, 256, 0, s>>>((const uint16_t*)in, in_ld, (uint16_t*)out,
                                                                            out_ld, R, C);
        }
        break;
      case 4: fast::tile_transpose_kernel<uint32_t, false><<<grid, 256, 0, s>>>((const uint32_t*)in, in_ld, (uint32_t*)out, out_ld, R, C); break;
      case 8: fast::tile_transpose_kernel<uint64_t, false><<<grid, 256, 0, s>>>((const uint64_t*)in, in_ld, (uint64_t*)out, out_ld, R, C); break;
      default: return 1;
    }
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
  }
  if (kind == 1) {
    // VNNI alpha 2 of an M x lcols 16-bit matrix: out (2M) x ceil(lcols/2)
    const int M = out_rows / 2;
    if (esize != 2 || alpha != 2 || M % 8 || in_ld % 8 || out_ld % 8 || reinterpret_cast<uintptr_t>(in) % 16 ||
        reinterpret_cast<uintptr_t>(out) % 16)
      return 1;
    const int64_t total = (int64_t)(M / 8) * out_cols;
    if (total == 0) return 0;
    fast::vnni2_kernel<<<grid_for(total), 256, 0, s>>>((const uint16_t*)in, in_ld, (uint16_t*)out, out_ld, M, lcols,
                                                        out_cols);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
  }
  if (kind == 2) {
    // VNNI(L, 2) -> VNNI(L^T, 2), 16-bit, even extents: an (lrows/2) x (lcols/2)
    // transpose of 8-byte 2x2 blocks (in block (h, g) = words (2h, g), (2h+1, g))
    if (esize != 2 || alpha != 2 || alpha_out != 2 || lrows % 2 || lcols % 2 || in_ld % 4 || out_ld % 4 ||
        reinterpret_cast<uintptr_t>(in) % 8 || reinterpret_cast<uintptr_t>(out) % 8)
      return 1;
    const int R = lrows / 2, C = lcols / 2;  // blocks: rows h (pairs of L rows), cols g (pairs of L cols)
    const unsigned grid = (unsigned)(((R + 31) / 32) * ((C + 31) / 32));
    if (grid == 0) return 0;
    // in block (h, g) at 8-byte index h + g * (in_ld / 4); out block (g, h) at g + h * (out_ld / 4)
    fast::tile_transpose_kernel<uint64_t, true><<<grid, 256, 0, s>>>((const uint64_t*)in, in_ld / 4, (uint64_t*)out,
                                                                     out_ld / 4, R, C);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
  }
  return 1;
}

int fast_dropout_inv(const DView& in, const uint8_t* mask, float scale, void* out, int out_dtype, int out_ld,
                     cudaStream_t s) {
  using namespace fast;
  const int rows = in.rows;
  if (rows % 8 || out_ld != rows || !dense(in, rows) || reinterpret_cast<uintptr_t>(out) % 16) return 1;
  if ((in.dtype != TPP_BF16 && in.dtype != TPP_FP32) || (out_dtype != TPP_BF16 && out_dtype != TPP_FP32)) return 1;
  const int64_t groups = (int64_t)rows / 8 * in.cols;
  if (groups == 0) return 0;
  const unsigned grid = grid_for(groups);
  if (in.dtype == TPP_BF16 && out_dtype == TPP_BF16)
    dropout_inv_vec_kernel<uint16_t, uint16_t><<<grid, 256, 0, s>>>(in.p, mask, scale, out, groups);
  else if (in.dtype == TPP_BF16)
    dropout_inv_vec_kernel<uint16_t, float><<<grid, 256, 0, s>>>(in.p, mask, scale, out, groups);
  else if (out_dtype == TPP_BF16)
    dropout_inv_vec_kernel<float, uint16_t><<<grid, 256, 0, s>>>(in.p, mask, scale, out, groups);
  else
    dropout_inv_vec_kernel<float, float><<<grid, 256, 0, s>>>(in.p, mask, scale, out, groups);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // namespace tpp

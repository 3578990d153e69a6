// C ABI (include/tpp_b200.h): argument validation mirroring the reference's
// exceptions, then dispatch to the sm_100a kernels.  No allocation and no
// host synchronisation on any path except where a reference call needs a
// scratch vector (reduce ALL), which comes from a cached device buffer.

#include <cstdio>
#include <mutex>
#include <string>

#include "common.cuh"

namespace tpp {

static thread_local std::string g_last_error;
static thread_local std::string g_last_config;

void set_last_config(const std::string& cfg) { g_last_config = cfg; }

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}
int cuda_status(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return TPP_E_CUDA;
}

static cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static int acc_dtype_of(int in) {
  if (in == TPP_FP64) return TPP_FP64;
  if (in == TPP_INT8) return TPP_INT32;
  return TPP_FP32;
}

// contraction.py:58-73 (GemmSpec.__post_init__)
static int check_gemm(const tpp_gemm_desc* d) {
  TPP_REQUIRE(d != nullptr, TPP_E_TENSOR, "null GEMM descriptor");
  TPP_REQUIRE(d->m >= 1 && d->n >= 1 && d->k >= 1, TPP_E_TENSOR, "GEMM extents must be positive");
  TPP_REQUIRE(d->in_dtype == TPP_FP64 || d->in_dtype == TPP_FP32 || d->in_dtype == TPP_BF16 ||
                  d->in_dtype == TPP_INT8,
              TPP_E_TENSOR, "unsupported input dtype");
  TPP_REQUIRE(d->out_dtype == acc_dtype_of(d->in_dtype), TPP_E_TENSOR,
              "output dtype must be the accumulator dtype for the input dtype");
  TPP_REQUIRE(d->a_vnni || d->lda >= d->m, TPP_E_TENSOR, "lda < M");
  TPP_REQUIRE(d->ldb >= d->k, TPP_E_TENSOR, "ldb < K");
  TPP_REQUIRE(d->ldc >= d->m, TPP_E_TENSOR, "ldc < M");
  TPP_REQUIRE(d->compute_path == 0 || d->in_dtype == TPP_BF16, TPP_E_TENSOR,
              "EMULATED_SPLIT applies to BF16 inputs");
  TPP_REQUIRE(!d->a_vnni || d->in_dtype == TPP_BF16 || d->in_dtype == TPP_INT8, TPP_E_TENSOR,
              "VNNI A layout needs a 16- or 8-bit input dtype");
  TPP_REQUIRE(d->engine != TPP_ENGINE_TENSOR || d->in_dtype == TPP_INT8 || d->in_dtype == TPP_BF16,
              TPP_E_UNSUPPORTED, "the tensor-core engine serves BF16 and INT8 inputs (FP32/FP64: ordered engine)");
  return TPP_OK;
}

static OrderedParams base_params(const tpp_gemm_desc* d, void* c) {
  OrderedParams p{};
  p.m = d->m;
  p.n = d->n;
  p.k = d->k;
  p.lda = d->lda;
  p.ldb = d->ldb;
  p.ldc = d->ldc;
  p.vnni = d->a_vnni;
  p.alpha = d->in_dtype == TPP_INT8 ? 4 : 2;
  p.c = reinterpret_cast<char*>(c);
  p.instances = 1;
  p.beta = d->beta;
  return p;
}

}  // namespace tpp

using namespace tpp;

extern "C" {

const char* tpp_last_error(void) { return g_last_error.c_str(); }
const char* tpp_last_config(void) { return g_last_config.c_str(); }

int tpp_debug_phase_timestamps(uint64_t* dev_buf) {
  set_debug_timestamps(reinterpret_cast<unsigned long long*>(dev_buf));
  return TPP_OK;
}
int tpp_set_tile_scheduling(int32_t mode) { return set_tile_scheduling(mode); }
int tpp_version(void) { return 1; }
int tpp_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

int tpp_brgemm_stride(const tpp_gemm_desc* d, const void* a, const void* b, int64_t stride_a,
                      int64_t stride_b, int64_t count, void* c, void* stream) {
  int rc = check_gemm(d);
  if (rc) return rc;
  TPP_REQUIRE(count >= 0, TPP_E_TENSOR, "negative batch count");
  // INT8: integer sums are order-independent, so the tcgen05 kind::i8 engine
  // is bitwise the reference (plain A, 16-byte aligned strides)
  if (d->in_dtype == TPP_INT8 && d->engine != TPP_ENGINE_ORDERED) {
    if (count == 0) {
      TPP_REQUIRE(d->engine != TPP_ENGINE_TENSOR, TPP_E_UNSUPPORTED, "INT8 tensor engine needs a non-empty batch");
    } else if (!d->a_vnni) {
      const int r = brgemm_i8_stride_tc(d->m, d->n, d->k, reinterpret_cast<const int8_t*>(a), d->lda,
                                        reinterpret_cast<const int8_t*>(b), d->ldb, stride_a, stride_b, count,
                                        reinterpret_cast<int32_t*>(c), d->ldc, d->beta, as_stream(stream));
      if (r != 1) return r;
    }
    TPP_REQUIRE(d->engine != TPP_ENGINE_TENSOR, TPP_E_UNSUPPORTED,
                "INT8 tensor engine: plain A and 16-byte aligned pointers / lda / ldb / strides");
  }
  // BF16: the tcgen05 BRGEMM (AUTO and TENSOR); ORDERED keeps the reference order
  if (d->in_dtype == TPP_BF16 && d->engine != TPP_ENGINE_ORDERED) {
    const int r = brgemm_grouped_tc(d, 0, a, b, stride_a, stride_b, nullptr, nullptr, count, c, nullptr, 1,
                                    as_stream(stream));
    if (r != 1) return r;
    TPP_REQUIRE(d->engine != TPP_ENGINE_TENSOR, TPP_E_UNSUPPORTED, "BF16 tensor engine: needs count >= 1");
  }
  OrderedParams p = base_params(d, c);
  p.mode = 0;
  p.count = count;
  p.a = reinterpret_cast<const char*>(a);
  p.b = reinterpret_cast<const char*>(b);
  p.stride_a = stride_a;
  p.stride_b = stride_b;
  return launch_brgemm_ordered(p, d->in_dtype, as_stream(stream));
}

int tpp_brgemm_offset(const tpp_gemm_desc* d, const void* a, const void* b,
                      const int64_t* a_offsets, const int64_t* b_offsets, int64_t count, void* c,
                      void* stream) {
  int rc = check_gemm(d);
  if (rc) return rc;
  TPP_REQUIRE(count >= 0, TPP_E_TENSOR, "negative batch count");
  TPP_REQUIRE(count == 0 || (a_offsets && b_offsets), TPP_E_TENSOR, "null offset arrays");
  // BF16 (AUTO / TENSOR): the tcgen05 BRGEMM (misaligned blocks take its
  // element-wise staging path, checked per stage on the device)
  if (d->engine != TPP_ENGINE_ORDERED && d->in_dtype == TPP_BF16) {
    const int r = brgemm_grouped_tc(d, 1, a, b, 0, 0, a_offsets, b_offsets, count, c, nullptr, 1, as_stream(stream));
    if (r != 1) return r;
    TPP_REQUIRE(d->engine != TPP_ENGINE_TENSOR, TPP_E_UNSUPPORTED, "BF16 tensor engine: needs count >= 1");
  }
  TPP_REQUIRE(d->engine != TPP_ENGINE_TENSOR, TPP_E_UNSUPPORTED, "tensor engine for OFFSET batches: BF16 inputs");
  OrderedParams p = base_params(d, c);
  p.mode = 1;
  p.count = count;
  p.a = reinterpret_cast<const char*>(a);
  p.b = reinterpret_cast<const char*>(b);
  p.a_offs = a_offsets;
  p.b_offs = b_offsets;
  return launch_brgemm_ordered(p, d->in_dtype, as_stream(stream));
}

int tpp_brgemm_address(const tpp_gemm_desc* d, const void* const* a_ptrs,
                       const void* const* b_ptrs, int64_t count, void* c, void* stream) {
  int rc = check_gemm(d);
  if (rc) return rc;
  TPP_REQUIRE(count >= 0, TPP_E_TENSOR, "negative batch count");
  TPP_REQUIRE(count == 0 || (a_ptrs && b_ptrs), TPP_E_TENSOR, "null pointer arrays");
  if (d->engine != TPP_ENGINE_ORDERED && d->in_dtype == TPP_BF16) {  // as tpp_brgemm_offset
    const int r = brgemm_grouped_tc(d, 2, nullptr, nullptr, 0, 0, reinterpret_cast<const int64_t*>(a_ptrs),
                                    reinterpret_cast<const int64_t*>(b_ptrs), count, c, nullptr, 1, as_stream(stream));
    if (r != 1) return r;
    TPP_REQUIRE(d->engine != TPP_ENGINE_TENSOR, TPP_E_UNSUPPORTED, "BF16 tensor engine: needs count >= 1");
  }
  TPP_REQUIRE(d->engine != TPP_ENGINE_TENSOR, TPP_E_UNSUPPORTED, "tensor engine for ADDRESS batches: BF16 inputs");
  OrderedParams p = base_params(d, c);
  p.mode = 2;
  p.count = count;
  p.a_ptrs = a_ptrs;
  p.b_ptrs = b_ptrs;
  return launch_brgemm_ordered(p, d->in_dtype, as_stream(stream));
}

int tpp_brgemm_grouped(const tpp_gemm_desc* d, int32_t kind, const void* a, const void* b, int64_t stride_a,
                       int64_t stride_b, const int64_t* a_index, const int64_t* b_index, int64_t count, void* c,
                       const int64_t* c_offsets, int64_t groups, void* stream) {
  int rc = check_gemm(d);
  if (rc) return rc;
  TPP_REQUIRE(kind >= 0 && kind <= 2, TPP_E_TENSOR, "batch kind must be 0 STRIDE, 1 OFFSET or 2 ADDRESS");
  TPP_REQUIRE(count >= 1 && groups >= 0, TPP_E_TENSOR, "grouped BRGEMM needs count >= 1");
  TPP_REQUIRE(groups <= 1 || c_offsets, TPP_E_TENSOR, "several groups need per-group C offsets");
  TPP_REQUIRE(kind == 0 || (a_index && b_index), TPP_E_TENSOR, "null offset / pointer arrays");
  TPP_REQUIRE(d->engine != TPP_ENGINE_ORDERED && d->in_dtype == TPP_BF16, TPP_E_UNSUPPORTED,
              "grouped BRGEMM runs the BF16 tensor-core engine (other dtypes: one brgemm call per group)");
  if (groups == 0) return TPP_OK;
  const int r = brgemm_grouped_tc(d, kind, a, b, stride_a, stride_b, a_index, b_index, count, c, c_offsets, groups,
                                  as_stream(stream));
  if (r != 1) return r;
  return fail(TPP_E_UNSUPPORTED, "grouped BRGEMM: BF16 inputs and count >= 1");
}

int tpp_brgemm_grouped_gang(const tpp_gemm_desc* d, int32_t kind, const void* a, const void* b, int64_t stride_a,
                            int64_t stride_b, const int64_t* a_index, const int64_t* b_index, int64_t count,
                            void* c, const int64_t* c_offsets, int64_t groups, const int32_t* gang, int32_t ngangs,
                            int32_t gang_m, int32_t gang_n, void* stream) {
  int rc = check_gemm(d);
  if (rc) return rc;
  TPP_REQUIRE(kind >= 0 && kind <= 2, TPP_E_TENSOR, "batch kind must be 0 STRIDE, 1 OFFSET or 2 ADDRESS");
  TPP_REQUIRE(count >= 1 && groups >= 1 && c_offsets && gang && ngangs >= 1, TPP_E_TENSOR,
              "ganged grouped BRGEMM needs count >= 1, C offsets and a gang table");
  TPP_REQUIRE(kind == 0 || (a_index && b_index), TPP_E_TENSOR, "null offset / pointer arrays");
  TPP_REQUIRE(d->engine != TPP_ENGINE_ORDERED && d->in_dtype == TPP_BF16, TPP_E_UNSUPPORTED,
              "grouped BRGEMM runs the BF16 tensor-core engine");
  const int r = brgemm_grouped_tc(d, kind, a, b, stride_a, stride_b, a_index, b_index, count, c, c_offsets, groups,
                                  as_stream(stream), gang, ngangs, gang_m, gang_n);
  if (r != 1) return r;
  return fail(TPP_E_UNSUPPORTED, "grouped BRGEMM: BF16 inputs and count >= 1");
}

int tpp_brgemm_grouped_bf16(const tpp_gemm_desc* d, int32_t kind, const void* a, const void* b, int64_t stride_a,
                            int64_t stride_b, const int64_t* a_index, const int64_t* b_index, int64_t count,
                            void* c_bf16, const int64_t* c_offsets, int64_t groups, const int32_t* gang,
                            int32_t ngangs, int32_t gang_m, int32_t gang_n, int32_t col_period, int32_t col_keep,
                            void* stream) {
  int rc = check_gemm(d);
  if (rc) return rc;
  TPP_REQUIRE(kind >= 0 && kind <= 2, TPP_E_TENSOR, "batch kind must be 0 STRIDE, 1 OFFSET or 2 ADDRESS");
  TPP_REQUIRE(count >= 1 && groups >= 1 && c_bf16 && (groups == 1 || c_offsets), TPP_E_TENSOR,
              "grouped BRGEMM (BF16 out) needs count >= 1, an output and per-group C offsets");
  TPP_REQUIRE(kind == 0 || (a_index && b_index), TPP_E_TENSOR, "null offset / pointer arrays");
  TPP_REQUIRE(!gang || ngangs >= 1, TPP_E_TENSOR, "empty gang table");
  TPP_REQUIRE(col_period >= 1 && col_keep >= 1 && col_keep <= col_period, TPP_E_TENSOR,
              "column map: 1 <= col_keep <= col_period");
  TPP_REQUIRE(d->beta == 0.0, TPP_E_TENSOR, "BF16 output needs beta = 0");
  TPP_REQUIRE(d->engine != TPP_ENGINE_ORDERED && d->in_dtype == TPP_BF16, TPP_E_UNSUPPORTED,
              "grouped BRGEMM runs the BF16 tensor-core engine");
  const int r = brgemm_grouped_tc(d, kind, a, b, stride_a, stride_b, a_index, b_index, count, nullptr, c_offsets,
                                  groups, as_stream(stream), gang, gang ? ngangs : 0, gang ? gang_m : 1,
                                  gang ? gang_n : 1, c_bf16, col_period, col_keep);
  if (r != 1) return r;
  return fail(TPP_E_UNSUPPORTED, "grouped BRGEMM: BF16 inputs and count >= 1");
}

int tpp_brgemm_stride_batched(const tpp_gemm_desc* d, const void* a, const void* b,
                              int64_t stride_a, int64_t stride_b, int64_t count, void* c,
                              int64_t instances, int64_t inst_a, int64_t inst_b, int64_t inst_c,
                              void* stream) {
  int rc = check_gemm(d);
  if (rc) return rc;
  TPP_REQUIRE(count >= 0 && instances >= 0, TPP_E_TENSOR, "negative batch count");
  OrderedParams p = base_params(d, c);
  p.mode = 0;
  p.count = count;
  p.a = reinterpret_cast<const char*>(a);
  p.b = reinterpret_cast<const char*>(b);
  p.stride_a = stride_a;
  p.stride_b = stride_b;
  p.instances = instances;
  p.inst_a = inst_a;
  p.inst_b = inst_b;
  p.inst_c = inst_c;
  return launch_brgemm_ordered(p, d->in_dtype, as_stream(stream));
}

// ---- FC -----------------------------------------------------------------
static int check_fc(const tpp_fc_desc* d) {
  TPP_REQUIRE(d != nullptr, TPP_E_TENSOR, "null FC descriptor");
  TPP_REQUIRE(d->m_b >= 1 && d->n_b >= 1 && d->k_b >= 1 && d->bm >= 1 && d->bn >= 1 && d->bk >= 1,
              TPP_E_TENSOR, "FC blocking factors must be positive");
  TPP_REQUIRE(d->in_dtype == TPP_FP32 || d->in_dtype == TPP_BF16, TPP_E_SPEC_DTYPE,
              "FC input dtype must be FP32 or BF16");
  TPP_REQUIRE(d->activation >= TPP_ACT_NONE && d->activation <= TPP_ACT_GELU, TPP_E_SPEC_FLAG,
              "unknown activation");
  return TPP_OK;
}

int tpp_fc_backward_data(const tpp_fc_desc* d, const void* w_packed, const void* dout,
                         const void* relu_mask_in, void* din, void* stream) {
  int rc = check_fc(d);
  if (rc) return rc;
  TPP_REQUIRE(d->in_dtype == TPP_BF16, TPP_E_SPEC_DTYPE, "FC backward runs on BF16 operands");
  TPP_REQUIRE(w_packed && dout && din, TPP_E_TENSOR, "null FC operand");
  TPP_REQUIRE(!(d->flags & TPP_FC_RELU_INV) || relu_mask_in, TPP_E_TENSOR,
              "RELU_INV requires a recorded bitmask");
  TPP_REQUIRE(!(d->flags & (TPP_FC_BIAS | TPP_FC_RESIDUAL | TPP_FC_RELU_MASK)) &&
                  d->activation == TPP_ACT_NONE,
              TPP_E_SPEC_FLAG, "backward-data fuses only RELU_INV");
  return fc_gemm_tc(1, d, w_packed, dout, nullptr, nullptr, nullptr, din, nullptr, relu_mask_in,
                    as_stream(stream));
}

int tpp_fc_backward_weights(const tpp_fc_desc* d, const void* dout, const void* x, void* dw,
                            void* stream) {
  int rc = check_fc(d);
  if (rc) return rc;
  TPP_REQUIRE(d->in_dtype == TPP_BF16, TPP_E_SPEC_DTYPE, "FC backward runs on BF16 operands");
  TPP_REQUIRE(dout && x && dw, TPP_E_TENSOR, "null FC operand");
  TPP_REQUIRE(!(d->flags & ~(TPP_FC_OUT_FP32 | TPP_FC_DYNAMIC_TILES)) && d->activation == TPP_ACT_NONE,
              TPP_E_SPEC_FLAG, "backward-weights takes only the FP32-output flag");
  return fc_gemm_tc(2, d, nullptr, dout, x, nullptr, nullptr, dw, nullptr, nullptr, as_stream(stream));
}

int tpp_fc_backward_weights_sgd(const tpp_fc_desc* d, const void* dout, const void* x, uint16_t* w_hi,
                                uint16_t* w_lo, float lr, void* stream) {
  int rc = check_fc(d);
  if (rc) return rc;
  TPP_REQUIRE(d->in_dtype == TPP_BF16, TPP_E_SPEC_DTYPE, "FC backward runs on BF16 operands");
  TPP_REQUIRE(dout && x && w_hi && w_lo, TPP_E_TENSOR, "null FC operand");
  TPP_REQUIRE(w_hi != w_lo, TPP_E_TENSOR, "hi and lo halves must be distinct buffers");
  TPP_REQUIRE(reinterpret_cast<uintptr_t>(w_hi) % 16 == 0 && reinterpret_cast<uintptr_t>(w_lo) % 16 == 0,
              TPP_E_TENSOR, "split-master halves must be 16-byte aligned");
  TPP_REQUIRE(!(d->flags & ~(TPP_FC_OUT_FP32 | TPP_FC_SGD | TPP_FC_DYNAMIC_TILES)) && d->activation == TPP_ACT_NONE,
              TPP_E_SPEC_FLAG, "backward-weights-SGD takes no epilogue flags");
  tpp_fc_desc dd = *d;
  dd.flags = TPP_FC_OUT_FP32 | TPP_FC_SGD | (d->flags & TPP_FC_DYNAMIC_TILES);
  return fc_gemm_tc(2, &dd, nullptr, dout, x, nullptr, nullptr, w_hi, nullptr, nullptr, as_stream(stream), w_lo, lr);
}

int tpp_softmax_xent_blocked(int32_t n_b, int32_t m_b, int32_t bn, int32_t bm, const float* logits,
                             const int32_t* targets, float scale, void* dlogits, float* loss,
                             void* stream) {
  TPP_REQUIRE(n_b >= 1 && m_b >= 1 && bn >= 1 && bm >= 1, TPP_E_TENSOR, "bad blocking");
  TPP_REQUIRE(logits && targets && dlogits, TPP_E_TENSOR, "null operand");
  return launch_softmax_xent_blocked(n_b, m_b, bn, bm, logits, targets, scale, dlogits, loss,
                                     as_stream(stream));
}

int64_t tpp_fc_packed_weight_bytes(const tpp_fc_desc* d) {
  if (!d) return -1;
  return (int64_t)d->m_b * d->k_b * d->bm * d->bk * (d->in_dtype == TPP_BF16 ? 2 : 4);
}

int tpp_fc_pack_weights(const tpp_fc_desc* d, const void* w_vnni, void* w_packed, void* stream) {
  int rc = check_fc(d);
  if (rc) return rc;
  TPP_REQUIRE(d->in_dtype == TPP_BF16, TPP_E_SPEC_DTYPE, "weight packing is for BF16 VNNI weights");
  TPP_REQUIRE(d->bk % 2 == 0, TPP_E_TENSOR, "VNNI-2 weights need an even reduce block");
  BlockRemap ident{0, 0, 0, 0, 0};
  return launch_word_transpose_blocks(w_vnni, w_packed, d->bk / 2, d->bm,
                                      (int64_t)d->m_b * d->k_b, ident, as_stream(stream));
}

int tpp_fc_forward(const tpp_fc_desc* d, const void* w, const void* x, const void* bias,
                   const void* residual, void* out, void* relu_mask, void* stream) {
  int rc = check_fc(d);
  if (rc) return rc;
  TPP_REQUIRE(w && x && out, TPP_E_TENSOR, "null FC operand");
  TPP_REQUIRE(!(d->flags & TPP_FC_BIAS) || bias, TPP_E_TENSOR, "bias flag without bias");
  TPP_REQUIRE(!(d->flags & TPP_FC_RESIDUAL) || residual, TPP_E_TENSOR, "residual flag without residual");
  TPP_REQUIRE(!(d->flags & TPP_FC_RELU_MASK) || (relu_mask && d->activation == TPP_ACT_RELU),
              TPP_E_SPEC_FLAG, "ReLU bitmask needs RELU activation and a mask buffer");
  if (d->in_dtype == TPP_BF16) return fc_forward_tc(d, w, x, bias, residual, out, relu_mask, as_stream(stream));
  // FP32: kernels.py:300-329 exactly — per output block a stride BRGEMM over
  // k_b blocks in reference order (bitwise), activation applied after.
  TPP_REQUIRE(!(d->flags & (TPP_FC_BIAS | TPP_FC_RESIDUAL)) && d->activation != TPP_ACT_GELU,
              TPP_E_UNSUPPORTED, "FP32 fc_forward supports the reference's RELU/none only");
  // instances over (ib_n, ib_m): C block (n, m) at (n*m_b + m)*bn*bm; A offset
  // m*k_b*bk*bm; B offset n*k_b*bn*bk.  One launch per ib_n keeps the instance
  // strides affine.
  tpp_gemm_desc g{};
  g.m = d->bm;
  g.n = d->bn;
  g.k = d->bk;
  g.lda = d->bm;
  g.ldb = d->bk;
  g.ldc = d->bm;
  g.in_dtype = TPP_FP32;
  g.out_dtype = TPP_FP32;
  g.beta = 0.0;
  for (int ibn = 0; ibn < d->n_b; ++ibn) {
    OrderedParams p = base_params(&g, reinterpret_cast<float*>(out) + (int64_t)ibn * d->m_b * d->bn * d->bm);
    p.mode = 0;
    p.count = d->k_b;
    p.a = reinterpret_cast<const char*>(w);
    p.b = reinterpret_cast<const char*>(reinterpret_cast<const float*>(x) + (int64_t)ibn * d->k_b * d->bn * d->bk);
    p.stride_a = (int64_t)d->bk * d->bm;
    p.stride_b = (int64_t)d->bn * d->bk;
    p.instances = d->m_b;
    p.inst_a = (int64_t)d->k_b * d->bk * d->bm;
    p.inst_b = 0;
    p.inst_c = (int64_t)d->bn * d->bm;
    rc = launch_brgemm_ordered(p, TPP_FP32, as_stream(stream));
    if (rc) return rc;
  }
  if (d->activation == TPP_ACT_RELU) {
    const int rows = d->bm, cols = d->n_b * d->m_b * d->bn;
    DView v{out, rows, cols, rows, TPP_FP32, TPP_BCAST_NONE};
    DView none{nullptr, 0, 0, 0, 0, 0};
    return launch_unary(TPP_UN_RELU, v, none, out, TPP_FP32, rows,
                        (d->flags & TPP_FC_RELU_MASK) ? reinterpret_cast<uint8_t*>(relu_mask) : nullptr,
                        false, as_stream(stream));
  }
  return TPP_OK;
}

// ---- conv -----------------------------------------------------------------
static int check_conv(const tpp_conv_desc* d) {
  TPP_REQUIRE(d != nullptr, TPP_E_TENSOR, "null conv descriptor");
  TPP_REQUIRE(d->n >= 1 && d->c_b >= 1 && d->k_b >= 1 && d->h >= 1 && d->w >= 1 && d->r >= 1 &&
                  d->s >= 1 && d->pad >= 0,
              TPP_E_TENSOR, "conv extents must be positive");
  TPP_REQUIRE(d->bc == 64 && d->bk == 64, TPP_E_UNSUPPORTED, "tensor-core conv needs bc = bk = 64");
  return TPP_OK;
}

int64_t tpp_conv_packed_weight_bytes(const tpp_conv_desc* d) {
  if (!d) return -1;
  return (int64_t)d->k_b * d->c_b * d->r * d->s * d->bc * d->bk * 2;
}

int tpp_conv_pack_weights(const tpp_conv_desc* d, const void* w_vnni, void* w_packed,
                          int32_t bwd_data, void* stream) {
  int rc = check_conv(d);
  if (rc) return rc;
  if (!bwd_data) {
    BlockRemap rm{1, d->k_b, d->c_b, d->r, d->s};
    return launch_word_transpose_blocks(w_vnni, w_packed, d->bc / 2, d->bk,
                                        (int64_t)d->k_b * d->c_b * d->r * d->s, rm,
                                        as_stream(stream));
  }
  if (bwd_data == 2)
    return launch_pack_conv_bwd_vnni(w_vnni, w_packed, d->k_b, d->c_b, d->r, d->s, d->bc, d->bk, as_stream(stream));
  return launch_pack_conv_bwd(w_vnni, w_packed, d->k_b, d->c_b, d->r, d->s, d->bc, d->bk,
                              as_stream(stream));
}

int tpp_conv_pad(int32_t n, int32_t c_b, int32_t hi, int32_t wi, int32_t ho, int32_t wo, int32_t top,
                 int32_t left, int32_t dil, const void* in, void* out, void* stream) {
  TPP_REQUIRE(n >= 0 && c_b >= 0 && hi >= 1 && wi >= 1 && ho >= 0 && wo >= 0 && top >= 0 && left >= 0 && dil >= 1,
              TPP_E_TENSOR, "bad conv padding extents");
  TPP_REQUIRE(in && out, TPP_E_TENSOR, "null operand");
  TPP_REQUIRE(reinterpret_cast<uintptr_t>(in) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0,
              TPP_E_TENSOR, "conv padding needs 16-byte aligned buffers");
  return launch_conv_pad(in, out, (int64_t)n * c_b, hi, wi, ho, wo, top, left, dil, as_stream(stream));
}

int tpp_conv_forward(const tpp_conv_desc* d, const void* w_packed, const void* x, void* out,
                     void* stream) {
  int rc = check_conv(d);
  if (rc) return rc;
  return conv_forward_tc(d->n, d->c_b, d->k_b, d->h, d->w, d->r, d->s, d->pad, w_packed, x, out,
                         as_stream(stream));
}

int tpp_conv_backward_data(const tpp_conv_desc* d, const void* w_packed_bwd, const void* dout,
                           void* din, void* stream) {
  int rc = check_conv(d);
  if (rc) return rc;
  // dI = conv(dO, flip(W)^T): input channels K_b*bk, output channels C_b*bc
  return conv_forward_tc(d->n, d->k_b, d->c_b, d->h, d->w, d->r, d->s, d->pad, w_packed_bwd, dout,
                         din, as_stream(stream));
}

int64_t tpp_conv_backward_weights_workspace_bytes(const tpp_conv_desc* d) {
  if (!d || check_conv(d)) return -1;
  return conv_dw_workspace_bytes(d->k_b, d->c_b, d->r, d->s);
}

int tpp_conv_backward_weights(const tpp_conv_desc* d, const void* x, const void* dout, float* dw,
                              void* workspace, void* stream) {
  int rc = check_conv(d);
  if (rc) return rc;
  TPP_REQUIRE(x && dout && dw && workspace, TPP_E_TENSOR, "conv backward-weights: null buffer");
  return conv_backward_weights_tc(d->n, d->c_b, d->k_b, d->h, d->w, d->r, d->s, d->pad, x, dout, dw, workspace,
                                  as_stream(stream));
}

// ---- eltwise ----------------------------------------------------------------
static bool valid_view(const tpp_tensor_desc* d) {
  if (!d || d->rows < 1 || d->cols < 1 || d->ld < 1) return false;
  if (d->bcast == TPP_BCAST_NONE && d->dtype != TPP_BIT && d->ld < d->rows) return false;
  return true;
}
static DView dview(const tpp_tensor_desc* d, const void* p) {
  DView v{p, d->rows, d->cols, d->ld, d->dtype, d->bcast};
  return v;
}
static bool is_float(int dt) { return dt == TPP_FP32 || dt == TPP_BF16 || dt == TPP_FP64; }

int tpp_unary(int32_t kind, const tpp_tensor_desc* in_d, const void* inp, const void* aux,
              const tpp_tensor_desc* out_d, void* out, void* mask_out, void* stream) {
  TPP_REQUIRE(valid_view(out_d), TPP_E_TENSOR, "bad output descriptor");
  if (kind == TPP_UN_ZERO) {
    TPP_REQUIRE(out_d->bcast == TPP_BCAST_NONE, TPP_E_TENSOR, "ZERO into a broadcast view");
    DView o = dview(out_d, out);
    return launch_unary(TPP_UN_ZERO, o, o, out, out_d->dtype, out_d->ld, nullptr,
                        out_d->dtype == TPP_FP64, as_stream(stream));
  }
  TPP_REQUIRE(valid_view(in_d), TPP_E_TENSOR, "bad input descriptor");
  TPP_REQUIRE(kind >= TPP_UN_IDENTITY && kind <= TPP_UN_GELU_INV, TPP_E_SPEC_FLAG, "unhandled unary kind");
  TPP_REQUIRE(in_d->rows == out_d->rows && in_d->cols == out_d->cols, TPP_E_TENSOR,
              "unary output shape mismatch");
  TPP_REQUIRE(is_float(in_d->dtype) && is_float(out_d->dtype), TPP_E_UNSUPPORTED,
              "GPU unary TPPs cover FP32/BF16/FP64");
  const bool f64 = in_d->dtype == TPP_FP64 || out_d->dtype == TPP_FP64;
  TPP_REQUIRE(!(f64 && (kind == TPP_UN_EXP || kind == TPP_UN_GELU || kind == TPP_UN_GELU_INV)),
              TPP_E_UNSUPPORTED, "FP64 approximations are not on the GPU path");
  TPP_REQUIRE(kind != TPP_UN_RELU_INV || aux, TPP_E_TENSOR, "RELU_INV requires a recorded bitmask");
  TPP_REQUIRE(kind != TPP_UN_GELU_INV || aux, TPP_E_TENSOR,
              "backward kind requires the forward input");
  TPP_REQUIRE(out_d->bcast == TPP_BCAST_NONE, TPP_E_TENSOR, "output must not be a broadcast view");
  DView a = dview(in_d, aux);
  if (kind == TPP_UN_GELU_INV) a = dview(in_d, aux);
  return launch_unary(kind, dview(in_d, inp), a, out, out_d->dtype, out_d->ld,
                      kind == TPP_UN_RELU ? reinterpret_cast<uint8_t*>(mask_out) : nullptr, f64,
                      as_stream(stream));
}

// ---- PRNG / dropout (ops.py:195-236, 326-328, 378-382, 430-444) --------------
int tpp_prng_seed(uint64_t seed, int32_t ncols, uint32_t* state, void* stream) {
  TPP_REQUIRE(ncols >= 1 && state, TPP_E_TENSOR, "PrngState needs ncols >= 1 and a state buffer");
  return launch_prng_seed(seed, ncols, state, as_stream(stream));
}

static bool states_disjoint(const uint32_t* a, const uint32_t* b, int cols) {
  const uintptr_t n = (uintptr_t)4 * cols * sizeof(uint32_t);
  const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
  return x + n <= y || y + n <= x;
}

int tpp_prng_fill(const uint32_t* state_in, uint32_t* state_out, const tpp_tensor_desc* out_d,
                  float* out, void* stream) {
  TPP_REQUIRE(valid_view(out_d) && out_d->bcast == TPP_BCAST_NONE, TPP_E_TENSOR, "bad PRNG output");
  TPP_REQUIRE(out_d->dtype == TPP_FP32, TPP_E_SPEC_DTYPE, "PRNG output must be FP32");
  TPP_REQUIRE(state_in && state_out && states_disjoint(state_in, state_out, out_d->cols), TPP_E_SPEC_FLAG,
              "PRNG needs disjoint state_in / state_out buffers");
  DView o = dview(out_d, out);
  return launch_prng_tile(0, o, state_in, state_out, 0.0, out, TPP_FP32, out_d->ld, nullptr, out_d->rows,
                          out_d->cols, false, as_stream(stream));
}

int tpp_dropout(const tpp_tensor_desc* in_d, const void* inp, const uint32_t* state_in, uint32_t* state_out,
                double p, const tpp_tensor_desc* out_d, void* out, uint8_t* mask_out, void* stream) {
  TPP_REQUIRE(valid_view(in_d) && valid_view(out_d), TPP_E_TENSOR, "bad dropout descriptor");
  TPP_REQUIRE(in_d->rows == out_d->rows && in_d->cols == out_d->cols, TPP_E_TENSOR,
              "DROPOUT output shape mismatch");
  TPP_REQUIRE(out_d->bcast == TPP_BCAST_NONE, TPP_E_TENSOR, "output must not be a broadcast view");
  TPP_REQUIRE(is_float(in_d->dtype) && is_float(out_d->dtype), TPP_E_UNSUPPORTED,
              "GPU dropout covers FP32/BF16/FP64");
  TPP_REQUIRE(p >= 0.0 && p < 1.0, TPP_E_SPEC_FLAG, "dropout p must be in [0, 1)");
  TPP_REQUIRE(state_in && state_out && states_disjoint(state_in, state_out, in_d->cols), TPP_E_SPEC_FLAG,
              "DROPOUT needs disjoint state_in / state_out buffers");
  TPP_REQUIRE(mask_out, TPP_E_TENSOR, "DROPOUT needs a mask buffer");
  const bool f64 = in_d->dtype == TPP_FP64;
  return launch_prng_tile(1, dview(in_d, inp), state_in, state_out, p, out, out_d->dtype, out_d->ld, mask_out,
                          in_d->rows, in_d->cols, f64, as_stream(stream));
}

int tpp_dropout_inv(const tpp_tensor_desc* in_d, const void* inp, const uint8_t* mask, double p,
                    const tpp_tensor_desc* out_d, void* out, void* stream) {
  TPP_REQUIRE(valid_view(in_d) && valid_view(out_d), TPP_E_TENSOR, "bad dropout descriptor");
  TPP_REQUIRE(in_d->rows == out_d->rows && in_d->cols == out_d->cols, TPP_E_TENSOR,
              "DROPOUT_INV output shape mismatch");
  TPP_REQUIRE(out_d->bcast == TPP_BCAST_NONE, TPP_E_TENSOR, "output must not be a broadcast view");
  TPP_REQUIRE(is_float(in_d->dtype) && is_float(out_d->dtype), TPP_E_UNSUPPORTED,
              "GPU dropout covers FP32/BF16/FP64");
  TPP_REQUIRE(mask, TPP_E_TENSOR, "DROPOUT_INV requires a recorded bitmask in secondary");
  return launch_dropout_inv(dview(in_d, inp), mask, p, out, out_d->dtype, out_d->ld, in_d->dtype == TPP_FP64,
                            as_stream(stream));
}

// ---- QUANTIZE / DEQUANTIZE (ops.py:447-469) -----------------------------------
int tpp_quantize(const tpp_tensor_desc* in_d, const float* inp, int32_t has_scale, double scale,
                 const tpp_tensor_desc* out_d, int8_t* out, void* workspace, double* scale_out, void* stream) {
  TPP_REQUIRE(valid_view(in_d) && valid_view(out_d), TPP_E_TENSOR, "bad quantize descriptor");
  TPP_REQUIRE(in_d->dtype == TPP_FP32 && out_d->dtype == TPP_INT8, TPP_E_SPEC_DTYPE, "QUANTIZE is FP32 -> INT8");
  TPP_REQUIRE(in_d->rows == out_d->rows && in_d->cols == out_d->cols, TPP_E_TENSOR,
              "QUANTIZE output shape mismatch");
  TPP_REQUIRE(out_d->bcast == TPP_BCAST_NONE, TPP_E_TENSOR, "output must not be a broadcast view");
  TPP_REQUIRE(has_scale || workspace, TPP_E_TENSOR, "QUANTIZE without a scale needs a 4-byte workspace");
  return launch_quantize(dview(in_d, inp), has_scale, scale, out, out_d->ld,
                         reinterpret_cast<uint32_t*>(workspace), scale_out, as_stream(stream));
}

int tpp_dequantize(const tpp_tensor_desc* in_d, const int8_t* inp, double scale, const tpp_tensor_desc* out_d,
                   float* out, void* stream) {
  TPP_REQUIRE(valid_view(in_d) && valid_view(out_d), TPP_E_TENSOR, "bad dequantize descriptor");
  TPP_REQUIRE(in_d->dtype == TPP_INT8 && out_d->dtype == TPP_FP32, TPP_E_SPEC_DTYPE, "DEQUANTIZE is INT8 -> FP32");
  TPP_REQUIRE(in_d->rows == out_d->rows && in_d->cols == out_d->cols, TPP_E_TENSOR,
              "DEQUANTIZE output shape mismatch");
  TPP_REQUIRE(out_d->bcast == TPP_BCAST_NONE, TPP_E_TENSOR, "output must not be a broadcast view");
  return launch_dequantize(dview(in_d, inp), scale, out, out_d->ld, as_stream(stream));
}

static int join_check(const tpp_tensor_desc* const* ds, int n, int* rows, int* cols) {
  int r = 0, c = 0;
  for (int i = 0; i < n; ++i) {
    r = r > ds[i]->rows ? r : ds[i]->rows;
    c = c > ds[i]->cols ? c : ds[i]->cols;
  }
  for (int i = 0; i < n; ++i) {
    // a logical view of a broadcast desc already has the full shape; a
    // physical 1xN / Mx1 without bcast may also join (ops.py:260-266)
    if (!(ds[i]->rows == 1 || ds[i]->rows == r) || !(ds[i]->cols == 1 || ds[i]->cols == c))
      return fail(TPP_E_TENSOR, "cannot broadcast-join operand shapes");
  }
  *rows = r;
  *cols = c;
  return TPP_OK;
}

static DView joined(const tpp_tensor_desc* d, const void* p, int rows, int cols) {
  DView v = dview(d, p);
  if (v.bcast == TPP_BCAST_NONE) {
    // implicit numpy broadcast of a physical 1 x N / M x 1 / 1 x 1 operand
    if (d->rows == 1 && d->cols == 1 && (rows > 1 || cols > 1)) v.bcast = TPP_BCAST_SCALAR;
    else if (d->rows == 1 && rows > 1) v.bcast = TPP_BCAST_ROW;
    else if (d->cols == 1 && cols > 1) v.bcast = TPP_BCAST_COL;
  }
  return v;
}

int tpp_binary(int32_t kind, const tpp_tensor_desc* a_d, const void* a,
               const tpp_tensor_desc* b_d, const void* b, const tpp_tensor_desc* out_d, void* out,
               void* stream) {
  TPP_REQUIRE(valid_view(a_d) && valid_view(b_d) && valid_view(out_d), TPP_E_TENSOR, "bad descriptor");
  TPP_REQUIRE(kind >= TPP_BIN_ADD && kind <= TPP_BIN_MIN, TPP_E_SPEC_FLAG, "unhandled binary kind");
  TPP_REQUIRE(is_float(a_d->dtype) && is_float(b_d->dtype) && is_float(out_d->dtype),
              TPP_E_UNSUPPORTED, "GPU binary TPPs cover FP32/BF16/FP64");
  const tpp_tensor_desc* ds[2] = {a_d, b_d};
  int rows, cols;
  int rc = join_check(ds, 2, &rows, &cols);
  if (rc) return rc;
  TPP_REQUIRE(out_d->rows == rows && out_d->cols == cols, TPP_E_TENSOR, "binary output shape mismatch");
  const bool f64 = a_d->dtype == TPP_FP64 || b_d->dtype == TPP_FP64;
  DView none{nullptr, 0, 0, 0, 0, 0};
  return launch_nary(2, kind, joined(a_d, a, rows, cols), joined(b_d, b, rows, cols), none, out,
                     rows, cols, out_d->dtype, out_d->ld, f64, as_stream(stream));
}

int tpp_ternary(int32_t kind, const tpp_tensor_desc* a_d, const void* a,
                const tpp_tensor_desc* b_d, const void* b, const tpp_tensor_desc* c_d,
                const void* c, const tpp_tensor_desc* out_d, void* out, void* stream) {
  TPP_REQUIRE(valid_view(a_d) && valid_view(b_d) && valid_view(c_d) && valid_view(out_d),
              TPP_E_TENSOR, "bad descriptor");
  TPP_REQUIRE(kind == TPP_TER_MULADD || kind == TPP_TER_NMULADD, TPP_E_SPEC_FLAG,
              "GEMM/BRGEMM live in the gemm module");
  TPP_REQUIRE(is_float(a_d->dtype) && is_float(b_d->dtype) && is_float(c_d->dtype) &&
                  is_float(out_d->dtype),
              TPP_E_UNSUPPORTED, "GPU ternary TPPs cover FP32/BF16/FP64");
  const tpp_tensor_desc* ds[3] = {a_d, b_d, c_d};
  int rows, cols;
  int rc = join_check(ds, 3, &rows, &cols);
  if (rc) return fail(TPP_E_SPEC_SHAPE, tpp_last_error());
  TPP_REQUIRE(out_d->rows == rows && out_d->cols == cols, TPP_E_TENSOR, "ternary output shape mismatch");
  const bool f64 = a_d->dtype == TPP_FP64 || b_d->dtype == TPP_FP64 || c_d->dtype == TPP_FP64;
  return launch_nary(3, kind, joined(a_d, a, rows, cols), joined(b_d, b, rows, cols),
                     joined(c_d, c, rows, cols), out, rows, cols, out_d->dtype, out_d->ld, f64,
                     as_stream(stream));
}

int tpp_reduce(const tpp_tensor_desc* in_d, const void* inp, int32_t axis, int32_t op,
               int32_t squared, const tpp_tensor_desc* out_d, void* out, void* stream) {
  TPP_REQUIRE(valid_view(in_d) && valid_view(out_d), TPP_E_TENSOR, "bad descriptor");
  TPP_REQUIRE(axis >= 0 && axis <= 2 && op >= 0 && op <= 3, TPP_E_SPEC_FLAG, "bad reduce spec");
  TPP_REQUIRE(is_float(in_d->dtype), TPP_E_UNSUPPORTED, "GPU reduce covers FP32/BF16/FP64");
  const int er = axis == 0 ? in_d->rows : 1;
  const int ec = axis == 1 ? in_d->cols : 1;
  TPP_REQUIRE(out_d->rows == er && out_d->cols == ec, TPP_E_TENSOR, "reduce output: wrong shape");
  const bool f64 = in_d->dtype == TPP_FP64;
  if (axis != 2)
    return launch_reduce(dview(in_d, inp), axis, op, squared, out, out_d->dtype, out_d->ld, nullptr, f64,
                         as_stream(stream));
  // ALL: per-column partials in a stream-ordered scratch vector (the pool
  // allocator: no device synchronisation, private to this call's stream
  // order, capturable in CUDA graphs)
  const cudaStream_t st = as_stream(stream);
  void* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, (size_t)in_d->cols * (f64 ? 8 : 4), st);
  if (e != cudaSuccess) return cuda_status(e, "cudaMallocAsync(reduce scratch)");
  const int rc = launch_reduce(dview(in_d, inp), axis, op, squared, out, out_d->dtype, out_d->ld, scratch, f64, st);
  e = cudaFreeAsync(scratch, st);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_status(e, "cudaFreeAsync(reduce scratch)");
  return TPP_OK;
}

int tpp_transform(int32_t kind, const tpp_tensor_desc* in_d, const void* inp, int32_t alpha,
                  int32_t alpha_out, int32_t rows, int32_t cols, const tpp_tensor_desc* out_d,
                  void* out, void* stream) {
  TPP_REQUIRE(valid_view(in_d) && valid_view(out_d), TPP_E_TENSOR, "bad descriptor");
  const int es = elem_size(in_d->dtype);
  TPP_REQUIRE(es > 0 && elem_size(out_d->dtype) == es, TPP_E_SPEC_DTYPE, "transform element size");
  if (kind == 0) {
    TPP_REQUIRE(out_d->rows == in_d->cols && out_d->cols == in_d->rows, TPP_E_TENSOR,
                "TRANSPOSE output: wrong shape");
    return launch_transform(0, es, inp, in_d->ld, out, out_d->rows, out_d->cols, out_d->ld, 0, 0, 0,
                            0, as_stream(stream));
  }
  if (kind == 1) {
    TPP_REQUIRE(alpha == (es == 2 ? 2 : (es == 1 ? 4 : -1)), TPP_E_SPEC_FLAG, "alpha incompatible with dtype");
    const int g = (in_d->cols + alpha - 1) / alpha;
    TPP_REQUIRE(out_d->rows == in_d->rows * alpha && out_d->cols == g, TPP_E_TENSOR,
                "VNNI output: wrong shape");
    return launch_transform(1, es, inp, in_d->ld, out, out_d->rows, out_d->cols, out_d->ld, alpha, 0,
                            in_d->rows, in_d->cols, as_stream(stream));
  }
  if (kind == 2) {
    const int want = es == 2 ? 2 : (es == 1 ? 4 : -1);
    TPP_REQUIRE(alpha == want && alpha_out == want, TPP_E_SPEC_FLAG, "alpha incompatible with dtype");
    TPP_REQUIRE(rows > 0 && cols > 0, TPP_E_SPEC_SHAPE, "VNNI_TO_VNNIT needs the logical extent");
    const int g = (rows + alpha_out - 1) / alpha_out;
    TPP_REQUIRE(out_d->rows == cols * alpha_out && out_d->cols == g, TPP_E_TENSOR,
                "VNNI_TO_VNNIT output: wrong shape");
    return launch_transform(2, es, inp, in_d->ld, out, out_d->rows, out_d->cols, out_d->ld, alpha,
                            alpha_out, rows, cols, as_stream(stream));
  }
  return fail(TPP_E_SPEC_FLAG, "unknown transform");
}

int tpp_convert(const tpp_tensor_desc* in_d, const void* inp, const tpp_tensor_desc* out_d,
                void* out, void* stream) {
  TPP_REQUIRE(valid_view(in_d) && valid_view(out_d), TPP_E_TENSOR, "bad descriptor");
  TPP_REQUIRE(in_d->bcast == TPP_BCAST_NONE, TPP_E_TENSOR, "convert requires a non-broadcast source");
  const int s = in_d->dtype, t = out_d->dtype;
  const bool ok = s == t || (s == TPP_FP32 && t == TPP_BF16) || (s == TPP_BF16 && t == TPP_FP32) ||
                  (s == TPP_FP32 && t == TPP_FP64) || (s == TPP_FP64 && t == TPP_FP32);
  TPP_REQUIRE(ok, TPP_E_TENSOR, "unsupported conversion");
  TPP_REQUIRE(in_d->rows == out_d->rows && in_d->cols == out_d->cols, TPP_E_TENSOR, "convert output mismatch");
  if (s == t && !is_float(s)) {
    return launch_transform(3, elem_size(s), inp, in_d->ld, out, out_d->rows, out_d->cols,
                            out_d->ld, 0, 0, 0, 0, as_stream(stream));
  }
  DView none{nullptr, 0, 0, 0, 0, 0};
  return launch_unary(TPP_UN_IDENTITY, dview(in_d, inp), none, out, t, out_d->ld, nullptr,
                      s == TPP_FP64 || t == TPP_FP64, as_stream(stream));
}

// ---- composite ----------------------------------------------------------------
int tpp_layernorm(const tpp_tensor_desc* x_d, const void* x, const tpp_tensor_desc* g_d,
                  const void* g, const tpp_tensor_desc* b_d, const void* b, double eps,
                  const tpp_tensor_desc* out_d, void* out, void* mean_out, void* var_out,
                  void* stream) {
  TPP_REQUIRE(valid_view(x_d) && valid_view(g_d) && valid_view(b_d) && valid_view(out_d),
              TPP_E_TENSOR, "bad descriptor");
  TPP_REQUIRE(x_d->cols >= 2, TPP_E_TENSOR, "layernorm needs a feature dimension of at least 2");
  TPP_REQUIRE(eps > 0, TPP_E_TENSOR, "eps must be positive");
  TPP_REQUIRE(g_d->rows == x_d->rows && g_d->cols == x_d->cols, TPP_E_TENSOR, "G must broadcast to the input shape");
  TPP_REQUIRE(b_d->rows == x_d->rows && b_d->cols == x_d->cols, TPP_E_TENSOR, "B must broadcast to the input shape");
  TPP_REQUIRE(out_d->rows == x_d->rows && out_d->cols == x_d->cols, TPP_E_TENSOR, "output shape mismatch");
  TPP_REQUIRE((x_d->dtype == TPP_FP32 || x_d->dtype == TPP_BF16) &&
                  (out_d->dtype == TPP_FP32 || out_d->dtype == TPP_BF16) &&
                  (g_d->dtype == TPP_FP32 || g_d->dtype == TPP_BF16) &&
                  (b_d->dtype == TPP_FP32 || b_d->dtype == TPP_BF16),
              TPP_E_UNSUPPORTED, "GPU layernorm covers FP32/BF16 views");
  DView xv{x, x_d->rows, x_d->cols, x_d->ld, x_d->dtype, x_d->bcast};
  DView gv{g, g_d->rows, g_d->cols, g_d->ld, g_d->dtype, g_d->bcast};
  DView bv{b, b_d->rows, b_d->cols, b_d->ld, b_d->dtype, b_d->bcast};
  return launch_layernorm_view(xv, gv, bv, eps, out, out_d->ld, out_d->dtype,
                               reinterpret_cast<float*>(mean_out), reinterpret_cast<float*>(var_out),
                               as_stream(stream));
}

int tpp_layernorm_blocked(int32_t n_b, int32_t m_b, int32_t bn, int32_t bm, int32_t dtype,
                          const void* x, const float* gamma, const float* beta, double eps,
                          void* out, float* mean_out, float* var_out, void* stream) {
  TPP_REQUIRE(n_b >= 1 && m_b >= 1 && bn >= 1 && bm >= 1, TPP_E_TENSOR, "bad blocking");
  TPP_REQUIRE(m_b * bm >= 2, TPP_E_TENSOR, "layernorm needs a feature dimension of at least 2");
  TPP_REQUIRE(eps > 0, TPP_E_TENSOR, "eps must be positive");
  TPP_REQUIRE(dtype == TPP_FP32 || dtype == TPP_BF16, TPP_E_SPEC_DTYPE, "dtype must be FP32 or BF16");
  TPP_REQUIRE(x && out, TPP_E_TENSOR, "null operand");
  return launch_layernorm_blocked(n_b, m_b, bn, bm, dtype, x, gamma, beta, eps, out, mean_out,
                                  var_out, as_stream(stream));
}

int tpp_layernorm_blocked_ex(int32_t n_b, int32_t m_b, int32_t bn, int32_t bm, int32_t dtype,
                             const void* x, const float* gamma, const float* beta, double eps,
                             void* out, float* mean_out, float* var_out, int32_t exact, void* stream) {
  TPP_REQUIRE(n_b >= 1 && m_b >= 1 && bn >= 1 && bm >= 1, TPP_E_TENSOR, "bad blocking");
  TPP_REQUIRE(m_b * bm >= 2, TPP_E_TENSOR, "layernorm needs a feature dimension of at least 2");
  TPP_REQUIRE(eps > 0, TPP_E_TENSOR, "eps must be positive");
  TPP_REQUIRE(dtype == TPP_FP32 || dtype == TPP_BF16, TPP_E_SPEC_DTYPE, "dtype must be FP32 or BF16");
  TPP_REQUIRE(x && out, TPP_E_TENSOR, "null operand");
  return launch_layernorm_blocked(n_b, m_b, bn, bm, dtype, x, gamma, beta, eps, out, mean_out,
                                  var_out, as_stream(stream), exact ? 1 : 0);
}

int tpp_softmax(int32_t s1, int32_t s2, int32_t s3, const tpp_tensor_desc* x_d, const void* x,
                const tpp_tensor_desc* y_d, void* y, void* stream) {
  TPP_REQUIRE(valid_view(x_d) && valid_view(y_d), TPP_E_TENSOR, "bad descriptor");
  TPP_REQUIRE(x_d->rows == s1 && x_d->cols == s2 * s3, TPP_E_TENSOR, "softmax input must be s1 x (s2*s3)");
  TPP_REQUIRE(y_d->rows == s1 && y_d->cols == s2 * s3, TPP_E_TENSOR, "softmax output shape mismatch");
  TPP_REQUIRE((x_d->dtype == TPP_FP32 || x_d->dtype == TPP_BF16) && y_d->dtype == TPP_FP32,
              TPP_E_UNSUPPORTED, "GPU softmax: FP32/BF16 in, FP32 out");
  DView xv{x, x_d->rows, x_d->cols, x_d->ld, x_d->dtype, x_d->bcast};
  return launch_softmax(s1, s2, s3, xv, reinterpret_cast<float*>(y), y_d->ld, as_stream(stream));
}

int tpp_split_sgd(int64_t n, uint16_t* hi, uint16_t* lo, const void* grad, int32_t grad_dtype,
                  float lr, void* stream) {
  TPP_REQUIRE(n >= 0, TPP_E_TENSOR, "negative size");
  TPP_REQUIRE(grad_dtype == TPP_FP32 || grad_dtype == TPP_BF16, TPP_E_SPEC_DTYPE, "grad dtype");
  return launch_split_sgd(n, hi, lo, grad, grad_dtype, lr, as_stream(stream));
}

}  // extern "C"

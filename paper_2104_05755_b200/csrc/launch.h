// Internal launch interfaces shared by the translation units of the library.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <mutex>
#include <map>
#include <set>
#include <utility>

#include "../../include/tpp_b200.h"

namespace tpp {

// programmatic dependent launch (PDL) for the library's kernels; TPP_NO_PDL=1
// switches it off (experiments: A/B of the launch overlap)
inline int pdl_allowed() {
  static const int v = getenv("TPP_NO_PDL") ? 0 : 1;
  return v;
}

// cudaFuncSetAttribute(max dynamic shared memory) per (kernel, device),
// raised whenever a launch needs more than the opt-in so far (kernels with a
// data-dependent footprint): thread-safe, and a second device used by the
// same process gets its own opt-in (the attribute is per device)
inline cudaError_t ensure_smem_attr(const void* kern, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  auto it = done.find({kern, dev});
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[{kern, dev}] = bytes;
  return e;
}

struct OrderedParams {
  int m, n, k, lda, ldb, ldc, vnni, alpha;
  int64_t count;
  int mode;  // 0 stride, 1 offset, 2 address
  const char* a;
  const char* b;
  int64_t stride_a, stride_b;
  const int64_t* a_offs;
  const int64_t* b_offs;
  const void* const* a_ptrs;
  const void* const* b_ptrs;
  char* c;
  int64_t inst_a, inst_b, inst_c;
  int64_t instances;
  double beta;
};
int launch_brgemm_ordered(const OrderedParams& p, int in_dtype, cudaStream_t s);

int fc_forward_tc(const tpp_fc_desc* d, const void* w_packed, const void* x, const void* bias,
                  const void* residual, void* out, void* mask, cudaStream_t stream);
int fc_gemm_tc(int flavor, const tpp_fc_desc* d, const void* w_packed, const void* x_or_dy,
               const void* x_for_dw, const void* bias, const void* residual, void* out,
               void* mask_out, const void* mask_in, cudaStream_t stream, uint16_t* sgd_lo = nullptr,
               float sgd_lr = 0.0f);
void set_debug_timestamps(unsigned long long* p);
int set_tile_scheduling(int mode);  // 0 flagged calls dynamic, 1 all, 2 none; other: query; returns the previous mode
unsigned long long* debug_timestamps();
// brgemm_grouped.cu (K11): BF16 BRGEMM on tcgen05 over stride / offset /
// address batches, `groups` C blocks per launch; 1 = not applicable
int brgemm_grouped_tc(const tpp_gemm_desc* d, int kind, const void* a, const void* b, int64_t stride_a,
                      int64_t stride_b, const int64_t* a_idx, const int64_t* b_idx, int64_t count, void* c,
                      const int64_t* c_off, int64_t groups, cudaStream_t s, const int32_t* gang = nullptr,
                      int ngangs = 0, int gang_ma = 1, int gang_nb = 1, void* c_bf16 = nullptr,
                      int col_period = 0, int col_keep = 0);
// brgemm_i8.cu (K10): INT8 STRIDE BRGEMM on tcgen05 kind::i8; 1 = not applicable
int brgemm_i8_stride_tc(int m, int n, int k, const int8_t* a, int64_t lda, const int8_t* b, int64_t ldb,
                        int64_t stride_a, int64_t stride_b, int64_t count, int32_t* c, int64_t ldc, double beta,
                        cudaStream_t s);
// 1-byte elements, 128-byte swizzle (INT8 BRGEMM operands)
int make_tma_map_5d_u8(CUtensorMap* m, const void* base, const uint64_t dims[5], const uint64_t strides[4],
                       const uint32_t box[5]);
// bf16 5-D TMA map (dims innermost first, byte strides of dims 1..4)
int make_tma_map_5d(CUtensorMap* m, const void* base, const uint64_t dims[5], const uint64_t strides[4],
                    const uint32_t box[5], int swizzle_bytes);
int launch_softmax_xent_blocked(int n_b, int m_b, int bn, int bm, const float* logits,
                                const int32_t* targets, float scale, void* dlogits, float* loss,
                                cudaStream_t s);
int64_t conv_dw_workspace_bytes(int Kb, int Cb, int R, int S);
int conv_backward_weights_tc(int N, int Cb, int Kb, int H, int W, int R, int S, int pad, const void* x,
                             const void* dout, float* dw, void* workspace, cudaStream_t stream);
int conv_forward_tc(int N, int Cb, int Kb, int H, int W, int R, int S, int pad,
                    const void* w_packed, const void* x, void* out, cudaStream_t stream);

struct BlockRemap {
  int mode;            // 0 identity, 1 conv fwd [Kb][Cb][R][S] -> [Kb][R][S][Cb]
  int d0, d1, d2, d3;  // src block index = ((i0*d1 + i1)*d2 + i2)*d3 + i3
};
int launch_word_transpose_blocks(const void* src, void* dst, int rows, int cols, int64_t nblocks,
                                 BlockRemap remap, cudaStream_t s);
int launch_pack_conv_bwd(const void* src, void* dst, int Kb, int Cb, int R, int S, int bc, int bk,
                         cudaStream_t s);
int launch_pack_conv_bwd_vnni(const void* src, void* dst, int Kb, int Cb, int R, int S, int bc, int bk,
                              cudaStream_t s);
int launch_conv_pad(const void* in, void* out, int64_t planes, int hi, int wi, int ho, int wo, int top, int left,
                    int dil, cudaStream_t s);
// kind: 0 TRANSPOSE, 1 VNNI, 2 VNNI_TO_VNNIT, 3 COPY
int launch_transform(int kind, int esize, const void* in, int in_ld, void* out, int out_rows,
                     int out_cols, int out_ld, int alpha, int alpha_out, int lrows, int lcols,
                     cudaStream_t s);

struct DView {
  const void* p;
  int rows, cols, ld, dtype, bcast;
};
// dense fast paths (eltwise_fast.cu): 0 handled, 1 not applicable, 2 launch error
int fast_dropout_inv(const DView& in, const uint8_t* mask, float scale, void* out, int out_dtype, int out_ld,
                     cudaStream_t s);
int fast_unary(int kind, const DView& in, const DView& aux, void* out, int out_dtype, int out_ld, uint8_t* mask_out,
               cudaStream_t s);
int fast_nary(int arity, int kind, const DView& a, const DView& b, const DView& c, void* out, int rows, int cols,
              int out_dtype, int out_ld, cudaStream_t s);
int fast_transform(int kind, int esize, const void* in, int in_ld, void* out, int out_rows, int out_cols,
                   int out_ld, int alpha, int alpha_out, int lrows, int lcols, cudaStream_t s);
// prng.cu (K8): xorshift128 streams, state SoA [4][cols]
int launch_prng_seed(uint64_t seed, int cols, uint32_t* state, cudaStream_t s);
int launch_prng_tile(int mode, const DView& in, const uint32_t* st_in, uint32_t* st_out, double p,
                     void* out, int out_dtype, int out_ld, uint8_t* mask_out, int rows, int cols, bool f64,
                     cudaStream_t s);
int launch_dropout_inv(const DView& in, const uint8_t* mask, double p, void* out, int out_dtype, int out_ld,
                       bool f64, cudaStream_t s);
// quant.cu (K9)
int launch_quantize(const DView& in, int has_scale, double scale, int8_t* out, int out_ld, uint32_t* amax_ws,
                    double* scale_out, cudaStream_t s);
int launch_dequantize(const DView& in, double scale, float* out, int out_ld, cudaStream_t s);
int launch_unary(int kind, const DView& in, const DView& aux, void* out, int out_dtype, int out_ld,
                 uint8_t* mask_out, bool f64, cudaStream_t s);
int launch_nary(int arity, int kind, const DView& a, const DView& b, const DView& c, void* out,
                int rows, int cols, int out_dtype, int out_ld, bool f64, cudaStream_t s);
int launch_reduce(const DView& in, int axis, int op, int squared, void* out, int out_dtype,
                  int out_ld, void* scratch, bool f64, cudaStream_t s);

int launch_layernorm_view(const DView& x, const DView& g, const DView& b, double eps, void* out,
                          int out_ld, int out_dtype, float* mean_out, float* var_out,
                          cudaStream_t s);
int launch_layernorm_blocked(int n_b, int m_b, int bn, int bm, int dtype, const void* x,
                             const float* gamma, const float* beta, double eps, void* out,
                             float* mean_out, float* var_out, cudaStream_t s, int exact = 1);
int launch_softmax(int s1, int s2, int s3, const DView& x, float* y, int y_ld, cudaStream_t s);
int launch_split_sgd(int64_t n, uint16_t* hi, uint16_t* lo, const void* grad, int grad_dtype,
                     float lr, cudaStream_t s);

}  // namespace tpp

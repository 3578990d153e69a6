/*
 * tpp_b200.h — C ABI of the B200-native (sm_100a) TPP BRGEMM hot path.
 *
 * Drop-in boundary for the reference operator API of "tensorprim"
 * (/root/reference/pkg/src/tensorprim).  The reference is pure Python/numpy
 * and has no FFI of its own; every entry point below replaces one Python
 * operator of that API (cited file:line) and is what a ctypes / cffi binding
 * of it binds.
 *
 * Conventions (mirroring the reference):
 *   - Memory-to-memory: every pointer is caller-owned DEVICE memory unless
 *     documented otherwise; the call writes outputs in place.
 *   - Tensors are column-major 2-D views (tensor.py:3-6): element (i, j) of a
 *     rows x cols view lives at i + j*ld.
 *   - Calls are stream-ordered and asynchronous (stream = cudaStream_t, may be
 *     NULL for the legacy default stream); no host sync, no allocation on the
 *     hot path.
 *   - Every function validates its arguments BEFORE launching anything and
 *     returns a tpp_status; tpp_last_error() gives the thread-local message.
 *     Status codes map to the reference exceptions: TPP_E_TENSOR ->
 *     TensorError (tensor.py:29), TPP_E_SPEC_* -> InvalidSpecError(code)
 *     (ops.py:174-179), TPP_E_INDEX -> IndexError.
 */
#ifndef TPP_B200_H
#define TPP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status / dtypes -------------------------------------------------- */
enum tpp_status {
  TPP_OK = 0,
  TPP_E_TENSOR = 1,       /* TensorError: shape / dtype / ld / alias / buffer   */
  TPP_E_SPEC_SHAPE = 2,   /* InvalidSpecError("shape")                           */
  TPP_E_SPEC_DTYPE = 3,   /* InvalidSpecError("dtype")                           */
  TPP_E_SPEC_FLAG = 4,    /* InvalidSpecError("flag")                            */
  TPP_E_INDEX = 5,        /* IndexError                                          */
  TPP_E_CUDA = 6,         /* CUDA runtime / driver failure                       */
  TPP_E_UNSUPPORTED = 7   /* valid spec outside what the sm_100a kernels cover  */
};

/* dtypes.py:17-24 (DType), same order */
enum tpp_dtype { TPP_FP64 = 0, TPP_FP32 = 1, TPP_BF16 = 2, TPP_INT32 = 3,
                 TPP_INT16 = 4, TPP_INT8 = 5, TPP_BIT = 6 };

/* tensor.py:33-37 (Bcast) */
enum tpp_bcast { TPP_BCAST_NONE = 0, TPP_BCAST_ROW = 1, TPP_BCAST_COL = 2,
                 TPP_BCAST_SCALAR = 3 };

const char* tpp_last_error(void);
/* Thread-local description of the last tensor-core kernel this thread
 * launched: its template instantiation <BN,STAGES,KPS,RES,CG,MC>, grid and
 * tile counts (e.g. "brgemm_tc_kernel<256,3,2,0,2,1> grid=148 tiles=64x16").
 * Lets tests assert which kernel a dispatch really ran. */
const char* tpp_last_config(void);
int tpp_version(void);
/* number of SMs of the current device (0 if no device) */
int tpp_device_sm_count(void);

/* ---- tensor descriptor: tensor.py:40-78 (TensorDesc) ------------------ */
typedef struct {
  int32_t rows, cols, ld;
  int32_t dtype;   /* tpp_dtype */
  int32_t bcast;   /* tpp_bcast */
} tpp_tensor_desc;

/* ---- BRGEMM TPP: contraction.py:44-85 (GemmSpec) --------------------- */
enum tpp_engine {
  TPP_ENGINE_AUTO = 0,     /* BF16 (STRIDE / OFFSET / ADDRESS, count >= 1) -> tcgen05
                              kind::f16 (normwise <= 2e-2); INT8 STRIDE -> tcgen05
                              kind::i8 (exact); everything else -> ordered         */
  TPP_ENGINE_ORDERED = 1,  /* SIMT, the reference's per-element order: bitwise parity  */
  TPP_ENGINE_TENSOR = 2    /* tcgen05.mma, TMEM accumulation: BF16 (all three batch
                              kinds; 16-byte aligned blocks with m, k, ldb, lda
                              multiples of 8 are staged with 16-byte copies, any
                              other block element-wise) and INT8 STRIDE, plain A  */
};

typedef struct {
  int32_t m, n, k, lda, ldb, ldc;
  int32_t in_dtype, out_dtype;  /* FP64->FP64, FP32->FP32, BF16->FP32, INT8->INT32 */
  int32_t a_vnni;               /* ALayout.VNNI: A is [ceil(K/alpha)][M][alpha]     */
  int32_t compute_path;         /* ComputePath: 0 NATIVE, 1 EMULATED_SPLIT          */
  int32_t engine;               /* tpp_engine                                        */
  int32_t reserved;
  double beta;                  /* C = beta*C + sum_i A_i B_i                        */
} tpp_gemm_desc;

/* contraction.py:261-322 brgemm() with BrgemmBatch.stride (contraction.py:162-168).
 * a, b: base pointers; strides and offsets are in ELEMENTS of in_dtype. */
int tpp_brgemm_stride(const tpp_gemm_desc* d, const void* a, const void* b,
                      int64_t stride_a, int64_t stride_b, int64_t count,
                      void* c, void* stream);
/* ... with BrgemmBatch.offset (contraction.py:152-160): device int64 offset arrays */
int tpp_brgemm_offset(const tpp_gemm_desc* d, const void* a, const void* b,
                      const int64_t* a_offsets, const int64_t* b_offsets, int64_t count,
                      void* c, void* stream);
/* ... with BrgemmBatch.address (contraction.py:144-150): device arrays of block pointers */
int tpp_brgemm_address(const tpp_gemm_desc* d, const void* const* a_ptrs,
                       const void* const* b_ptrs, int64_t count, void* c, void* stream);
/* Many independent BF16 BRGEMMs of one GemmSpec in ONE tcgen05 launch (the
 * GPU form of the reference's per-block job loops, kernels.py:312-329, and of
 * composing a layer from brgemm calls, contraction.py:261-322): group g
 * computes C_g = beta*C_g + sum_{i<count} A_{g,i} B_{g,i} with
 *   C_g = c + c_offsets[g] (elements; c_offsets may be NULL when groups == 1)
 *   kind 0 STRIDE:  A_{g,i} = a + (a_index ? a_index[g] : 0) + i*stride_a (b alike)
 *   kind 1 OFFSET:  A_{g,i} = a + a_index[g*count + i]              (b alike)
 *   kind 2 ADDRESS: A_{g,i} = ((const void* const*)a_index)[g*count + i]
 * All index arrays are device memory; engine AUTO or TENSOR, BF16 only, any
 * shape / alignment (16-byte aligned blocks with m, k, ldb, lda multiples of
 * 8 take the 16-byte staging path, others element-wise staging).
 * FP32 C, accumulated in TMEM over the whole batch (sum order differs from
 * the reference: <= 2e-2 normwise, north_star's BF16 tolerance). */
int tpp_brgemm_grouped(const tpp_gemm_desc* d, int32_t kind, const void* a, const void* b,
                       int64_t stride_a, int64_t stride_b, const int64_t* a_index,
                       const int64_t* b_index, int64_t count, void* c, const int64_t* c_offsets,
                       int64_t groups, void* stream);
/* tpp_brgemm_grouped with the groups tiled in gangs: gang j is gang_m (1 or
 * 2) x gang_n (1, 2, 4) groups where the groups of a gang row share their A
 * lists and those of a gang column their B lists (e.g. every C block of one
 * weight block row of an FC composition), so one tile loads each A and B
 * block once and runs M = 64 gang_m x N = 64 gang_n (or n, gang_n = 1) MMAs.
 * `gang` (device, int32) = rows [ngangs][gang_m] (a group whose A list feeds
 * the row), cols [ngangs][gang_n] (a group whose B list feeds the column),
 * cells [ngangs][gang_m][gang_n] (the group whose C a cell is), -1 = empty.
 * Needs m <= 64 (and n <= 64 for gang_n > 1).  Same results as the ungrouped
 * call (each C block is the same MMA chain over the same blocks). */
int tpp_brgemm_grouped_gang(const tpp_gemm_desc* d, int32_t kind, const void* a, const void* b,
                            int64_t stride_a, int64_t stride_b, const int64_t* a_index,
                            const int64_t* b_index, int64_t count, void* c, const int64_t* c_offsets,
                            int64_t groups, const int32_t* gang, int32_t ngangs, int32_t gang_m,
                            int32_t gang_n, void* stream);
/* tpp_brgemm_grouped(_gang) with the C blocks emitted in BF16 (beta = 0): the
 * FP32 accumulator of each element is narrowed RNE with the reference's NaN
 * rule (dtypes.py:82-97) -- the same bits as an FP32 call followed by
 * tpp_convert -- and block column v goes to column (v / col_period) *
 * col_keep + v % col_period of the output block at c_bf16 + c_offsets[g]
 * (column stride ldc), dropped when v % col_period >= col_keep.  This is the
 * conv composition's tail (kernels.py conv: padded-width rows of Wp virtual
 * columns, Q kept) fused into the BRGEMM epilogue; col_period = col_keep =
 * n keeps every column.  gang may be null (ungrouped tiling). */
int tpp_brgemm_grouped_bf16(const tpp_gemm_desc* d, int32_t kind, const void* a, const void* b,
                            int64_t stride_a, int64_t stride_b, const int64_t* a_index,
                            const int64_t* b_index, int64_t count, void* c_bf16, const int64_t* c_offsets,
                            int64_t groups, const int32_t* gang, int32_t ngangs, int32_t gang_m,
                            int32_t gang_n, int32_t col_period, int32_t col_keep, void* stream);
/* Many independent stride-BRGEMMs in one launch (the GPU form of the
 * reference's `threads=` job loop over disjoint C tiles, contraction.py:317-322
 * and kernels.py:323-329): instance j uses a + j*inst_a, b + j*inst_b,
 * c + j*inst_c (elements). */
int tpp_brgemm_stride_batched(const tpp_gemm_desc* d, const void* a, const void* b,
                              int64_t stride_a, int64_t stride_b, int64_t count,
                              void* c, int64_t instances, int64_t inst_a,
                              int64_t inst_b, int64_t inst_c, void* stream);

/* ---- blocked FC driver: kernels.py:287-329 (FcSpec / fc_forward) -------
 * Reference naming: A (weights) [m_b][k_b][bk][bm] (FP32) or VNNI
 * [m_b][k_b][bk/2][bm][2] (BF16); B (input) [n_b][k_b][bn][bk];
 * C (output) [n_b][m_b][bn][bm].  FP32 runs the reference order (bitwise);
 * BF16 runs tcgen05 with the epilogue TPPs fused into the GEMM tail. */
enum tpp_act { TPP_ACT_NONE = 0, TPP_ACT_RELU = 1, TPP_ACT_GELU = 2 };
enum tpp_fc_flags { TPP_FC_BIAS = 1, TPP_FC_RESIDUAL = 2, TPP_FC_RELU_MASK = 4,
                    TPP_FC_OUT_FP32 = 8, TPP_FC_BIAS_FP32 = 16, TPP_FC_RELU_INV = 32,
                    TPP_FC_SGD = 64,
                    /* draw this GEMM's tiles from a per-stream ticket counter instead of
                     * the static round-robin walk: for GEMMs the caller runs side by
                     * side on two streams (they fill each other's idle SMs) */
                    TPP_FC_DYNAMIC_TILES = 128 };

typedef struct {
  int32_t m_b, n_b, k_b, bm, bn, bk;
  int32_t in_dtype;     /* TPP_FP32 or TPP_BF16                                 */
  int32_t activation;   /* tpp_act                                              */
  int32_t flags;        /* tpp_fc_flags                                         */
  int32_t block_n;      /* tile width in output features for the TC kernel; 0=auto */
} tpp_fc_desc;

/* bytes of the packed (UMMA-canonical, K-major) weight buffer */
int64_t tpp_fc_packed_weight_bytes(const tpp_fc_desc* d);
/* VNNI weights -> K-major blocks [m_b][k_b][bm][bk] (a 32-bit word transpose
 * per block; transform VNNI_TO_VNNIT semantics, ops.py:556-565). */
int tpp_fc_pack_weights(const tpp_fc_desc* d, const void* w_vnni, void* w_packed,
                        void* stream);
/* out = act(W x + bias) + residual, narrowed to BF16 (RNE, dtypes.py:82-97)
 * unless TPP_FC_OUT_FP32.  bias: [m_b*bm]; residual/out: [n_b][m_b][bn][bm];
 * relu_mask: per-block column-major bitmask (tensor.py:238-261), i.e. bytes
 * [n_b][m_b][bn][ceil(bm/8)].  w: packed weights for BF16, plain A for FP32. */
int tpp_fc_forward(const tpp_fc_desc* d, const void* w, const void* x,
                   const void* bias, const void* residual, void* out, void* relu_mask,
                   void* stream);

/* Backward of the blocked FC (BF16, tcgen05), the training-side BRGEMMs of
 * PAPER.md:700-720 (kernel K8).  `d` describes the
 * FORWARD layer.  Both read the blocked buffers in place (MN-major UMMA
 * operands) — no transposed copies.
 *   backward-data:    din[n_b][k_b][bn][bk] = dout . W, then, with
 *                     TPP_FC_RELU_INV in d->flags, where(mask_in, ., 0)
 *                     (ops.py:367-369) with the forward input's ReLU bitmask
 *                     (layout of din, bytes [n_b][k_b][bn][bk/8]).
 *   backward-weights: dW[m_b][k_b][bm][bk] (packed weight layout) =
 *                     sum over tokens dout^T x; FP32 unless d->flags lacks
 *                     TPP_FC_OUT_FP32 (then BF16). */
int tpp_fc_backward_data(const tpp_fc_desc* d, const void* w_packed, const void* dout,
                         const void* relu_mask_in, void* din, void* stream);
int tpp_fc_backward_weights(const tpp_fc_desc* d, const void* dout, const void* x, void* dw,
                            void* stream);
/* Backward-weights with the split-SGD update fused into the GEMM epilogue
 * (kernels.py:235-251, single rank: no gradient exchange in between): the
 * FP32 dW tile is never stored; each element updates the split FP32 master
 * in place, W = hi:lo, W - dW*fp32(lr), re-split into w_hi (BF16 bits, the
 * packed weights the GEMMs read) and w_lo.  Bitwise equal to
 * tpp_fc_backward_weights (FP32) followed by tpp_split_sgd.  w_hi / w_lo:
 * [m_b][k_b][bm][bk], 16-byte aligned; no other GEMM may read w_hi while
 * this runs (issue the layer's backward-data first). */
int tpp_fc_backward_weights_sgd(const tpp_fc_desc* d, const void* dout, const void* x, uint16_t* w_hi,
                                uint16_t* w_lo, float lr, void* stream);
/* Softmax cross-entropy gradient on blocked FP32 logits [n_b][m_b][bn][bm]
 * (tokens x classes): per token the reference softmax (kernels.py:84-99 with
 * exp_taylor, approx.py:190-218), then dlogits = (p - onehot(target)) * scale
 * (BF16, same blocked layout) and loss[t] = -log(p[target]) (FP32). */
int tpp_softmax_xent_blocked(int32_t n_b, int32_t m_b, int32_t bn, int32_t bm, const float* logits,
                             const int32_t* targets, float scale, void* dlogits, float* loss,
                             void* stream);

/* ---- direct convolution via offset BRGEMM --------------
 * Input [N][C_b][H][W][bc], weights VNNI [K_b][C_b][R][S][bc/2][bk][2],
 * output [N][K_b][P][Q][bk]; stride 1, symmetric zero padding `pad`. */
typedef struct {
  int32_t n, c_b, k_b, h, w, r, s, pad, bc, bk;
  int32_t flags;        /* reserved */
  int32_t reserved;
} tpp_conv_desc;
int64_t tpp_conv_packed_weight_bytes(const tpp_conv_desc* d);
/* bwd_data=0: pack for forward; 1: flip taps and swap C/K (VNNI_TO_VNNIT per
 * tap) for backward-data, which is then a forward conv of dO; 2: the same
 * flipped / swapped weights kept in the reference VNNI layout
 * [C_b][K_b][R][S][bk/2][bc][2] (the generic offset-BRGEMM path's A blocks). */
int tpp_conv_pack_weights(const tpp_conv_desc* d, const void* w_vnni, void* w_packed,
                          int32_t bwd_data, void* stream);
int tpp_conv_forward(const tpp_conv_desc* d, const void* w_packed, const void* x,
                     void* out, void* stream);
/* Explicit zero padding / zero insertion of a blocked activation (the padded
 * input the reference's offset-BRGEMM convolution reads, kernels.py-style
 * composition): out[N][C_b][ho][wo][64](y, x) = in[N][C_b][hi][wi][64]
 * ((y - top) / dil, (x - left) / dil) when both divide and fall inside, else 0. */
int tpp_conv_pad(int32_t n, int32_t c_b, int32_t hi, int32_t wi, int32_t ho, int32_t wo, int32_t top,
                 int32_t left, int32_t dil, const void* in, void* out, void* stream);
/* dI[N][C_b][H][W][bc] from dO[N][K_b][P][Q][bk] with bwd-packed weights */
int tpp_conv_backward_data(const tpp_conv_desc* d, const void* w_packed_bwd,
                           const void* dout, void* din, void* stream);
/* Backward-weights (no reference kernel — the oracle is the
 * composition dW[k][c][r][s] = sum_{n,p,q} dO[n][k][p][q] * Xpad[n][c][p+r][q+s]):
 * dW FP32 [K_b][C_b][R][S][bc][bk] (element (c, k) of a tap at c*bk + k).
 * `workspace` holds per-CTA partials (tpp_conv_backward_weights_workspace_bytes);
 * they are summed in a fixed order, so results are deterministic. */
int64_t tpp_conv_backward_weights_workspace_bytes(const tpp_conv_desc* d);
int tpp_conv_backward_weights(const tpp_conv_desc* d, const void* x, const void* dout, float* dw,
                              void* workspace, void* stream);

/* ---- elementwise / reduce / transform TPPs (ops.py) -------------------- */
/* ops.py:32-64 UnaryKind subset implemented on the GPU */
enum tpp_unary {
  TPP_UN_IDENTITY = 0, TPP_UN_ZERO = 1, TPP_UN_SQUARE = 2, TPP_UN_INC = 3, TPP_UN_DEC = 4,
  TPP_UN_SQRT = 5, TPP_UN_RECIPROCAL = 6, TPP_UN_RSQRT = 7, TPP_UN_EXP = 8,
  TPP_UN_RELU = 9, TPP_UN_RELU_INV = 10, TPP_UN_GELU = 11, TPP_UN_GELU_INV = 12
};
/* ops.py:284-386 apply_unary.  aux: RELU_INV -> input bitmask (bytes),
 * GELU_INV -> forward input x (same desc as inp).  mask_out: RELU bitmask. */
int tpp_unary(int32_t kind, const tpp_tensor_desc* in_d, const void* inp, const void* aux,
              const tpp_tensor_desc* out_d, void* out, void* mask_out, void* stream);

/* ---- PRNG / dropout (ops.py:195-236 PrngState, 326-328 PRNG, 378-382
 * DROPOUT_INV, 430-444 DROPOUT).  A stream state is device memory holding
 * uint32 [4][ncols] (the x, y, z, w words of every column's xorshift128
 * stream).  Calls that advance a stream read state_in and write the advanced
 * stream to state_out; the two buffers must not overlap. */
/* PrngState(seed, ncols): splitmix64(seed ^ col) seeding, never all-zero */
int tpp_prng_seed(uint64_t seed, int32_t ncols, uint32_t* state, void* stream);
/* UnaryKind.PRNG: out (FP32, rows x cols) = uniform_block(rows) */
int tpp_prng_fill(const uint32_t* state_in, uint32_t* state_out, const tpp_tensor_desc* out_d,
                  float* out, void* stream);
/* UnaryKind.DROPOUT: keep = u >= float32(p); mask_out = keep bitmask
 * (tensor.py:246-254 layout); out = keep ? x * (1 / (1 - p)) : 0.  0 <= p < 1. */
int tpp_dropout(const tpp_tensor_desc* in_d, const void* inp, const uint32_t* state_in,
                uint32_t* state_out, double p, const tpp_tensor_desc* out_d, void* out,
                uint8_t* mask_out, void* stream);
/* UnaryKind.DROPOUT_INV: out = mask ? x * (1 / (1 - p)) : 0 (scale 0 if p >= 1) */
int tpp_dropout_inv(const tpp_tensor_desc* in_d, const void* inp, const uint8_t* mask, double p,
                    const tpp_tensor_desc* out_d, void* out, void* stream);

/* ---- QUANTIZE / DEQUANTIZE (ops.py:447-469), symmetric per-tensor INT8 ----
 * tpp_quantize: FP32 view -> INT8 (same logical shape).  has_scale = 0:
 * scale = max|x| / 127 (1.0 if that max is not > 0); else the given scale.
 * q = clip(rint(x / scale), -127, 127) in double, NaN -> 0.  workspace: 4
 * bytes of device memory; scale_out: device double receiving the scale used
 * (the reference's out.tertiary["scale"]). */
int tpp_quantize(const tpp_tensor_desc* in_d, const float* inp, int32_t has_scale, double scale,
                 const tpp_tensor_desc* out_d, int8_t* out, void* workspace, double* scale_out,
                 void* stream);
/* tpp_dequantize: INT8 view -> FP32, float32(q) * float32(scale) */
int tpp_dequantize(const tpp_tensor_desc* in_d, const int8_t* inp, double scale,
                   const tpp_tensor_desc* out_d, float* out, void* stream);

/* ops.py:66-75 BinaryKind elementwise subset */
enum tpp_binary { TPP_BIN_ADD = 0, TPP_BIN_SUB = 1, TPP_BIN_MUL = 2, TPP_BIN_DIV = 3,
                  TPP_BIN_MAX = 4, TPP_BIN_MIN = 5 };
/* ops.py:747-782 apply_binary (ROW/COL/SCALAR broadcast on either input) */
int tpp_binary(int32_t kind, const tpp_tensor_desc* a_d, const void* a,
               const tpp_tensor_desc* b_d, const void* b,
               const tpp_tensor_desc* out_d, void* out, void* stream);

enum tpp_ternary { TPP_TER_MULADD = 0, TPP_TER_NMULADD = 1 };
/* ops.py:796-816 apply_ternary MULADD (c + a*b) / NMULADD (c - a*b) */
int tpp_ternary(int32_t kind, const tpp_tensor_desc* a_d, const void* a,
                const tpp_tensor_desc* b_d, const void* b,
                const tpp_tensor_desc* c_d, const void* c,
                const tpp_tensor_desc* out_d, void* out, void* stream);

/* ops.py:484-522 reduce: axis 0 ROWS, 1 COLS, 2 ALL; op 0 SUM, 1 MUL, 2 MIN, 3 MAX */
int tpp_reduce(const tpp_tensor_desc* in_d, const void* inp, int32_t axis, int32_t op,
               int32_t squared, const tpp_tensor_desc* out_d, void* out, void* stream);

/* ops.py:537-570 transform: 0 TRANSPOSE, 1 VNNI (alpha), 2 VNNI_TO_VNNIT
 * (alpha, alpha_out, logical rows/cols of the pre-VNNI tensor) */
int tpp_transform(int32_t kind, const tpp_tensor_desc* in_d, const void* inp,
                  int32_t alpha, int32_t alpha_out, int32_t rows, int32_t cols,
                  const tpp_tensor_desc* out_d, void* out, void* stream);

/* tensor.py:328-355 convert (FP32<->BF16, FP32<->FP64, same-dtype copy) */
int tpp_convert(const tpp_tensor_desc* in_d, const void* inp,
                const tpp_tensor_desc* out_d, void* out, void* stream);

/* ---- composite kernels (kernels.py) ------------------------------------ */
/* kernels.py:134-176 layernorm on a column-major rows x cols view (each row
 * normalised over its columns).  g, b: views broadcastable to rows x cols.
 * mean_out / var_out: FP32 [rows] or NULL.  Bitwise to the reference. */
int tpp_layernorm(const tpp_tensor_desc* x_d, const void* x,
                  const tpp_tensor_desc* g_d, const void* g,
                  const tpp_tensor_desc* b_d, const void* b, double eps,
                  const tpp_tensor_desc* out_d, void* out, void* mean_out, void* var_out,
                  void* stream);
/* The same equation on the blocked activation layout [n_b][m_b][bn][bm]
 * (tokens x features, what fc_forward produces): every token is normalised
 * over its m_b*bm features in ascending feature order.  gamma/beta: [m_b*bm]
 * FP32 or NULL (1 / 0).  x/out dtype: TPP_FP32 or TPP_BF16. */
int tpp_layernorm_blocked(int32_t n_b, int32_t m_b, int32_t bn, int32_t bm, int32_t dtype,
                          const void* x, const float* gamma, const float* beta, double eps,
                          void* out, float* mean_out, float* var_out, void* stream);
/* exact = 1: as tpp_layernorm_blocked (the reference order, bitwise);
 * exact = 0: tolerance mode for BF16 (tree-ordered sums, FMA-contracted
 * scaling; within 1e-5 relative of the exact statistics) */
int tpp_layernorm_blocked_ex(int32_t n_b, int32_t m_b, int32_t bn, int32_t bm, int32_t dtype,
                             const void* x, const float* gamma, const float* beta, double eps,
                             void* out, float* mean_out, float* var_out, int32_t exact, void* stream);
/* kernels.py:84-99 softmax(SoftmaxSpec(s1, s2, s3)) on a FP32 s1 x (s2*s3) view */
int tpp_softmax(int32_t s1, int32_t s2, int32_t s3, const tpp_tensor_desc* x_d,
                const void* x, const tpp_tensor_desc* y_d, void* y, void* stream);
/* kernels.py:235-251 split_sgd_step: hi (BF16) / lo (INT16) halves updated
 * in place with W - grad*fp32(lr); grad FP32 or BF16, all contiguous, n elems */
int tpp_split_sgd(int64_t n, uint16_t* hi, uint16_t* lo, const void* grad,
                  int32_t grad_dtype, float lr, void* stream);

/* ---- diagnostics ------------------------------------------------------- */
/* When `dev_buf` (>= 8 uint64, device memory) is non-NULL, subsequent FC
 * tensor-core launches record %globaltimer phase stamps of CTA 0: start,
 * prologue done, first stage landed, last MMA issued, accumulator ready,
 * epilogue done, exit.  NULL disables.  Tools only. */
int tpp_debug_phase_timestamps(uint64_t* dev_buf);
/* Tile scheduling of the persistent tensor-core FC GEMMs: 0 = static
 * round-robin except calls flagged TPP_FC_DYNAMIC_TILES (the default), 1 =
 * dynamic for every call, 2 = static for every call (also TPP_STATIC_TILES=1
 * at startup), other values query.  Returns the previous mode.  Results do
 * not depend on it. */
int tpp_set_tile_scheduling(int32_t mode);

#ifdef __cplusplus
}
#endif
#endif /* TPP_B200_H */

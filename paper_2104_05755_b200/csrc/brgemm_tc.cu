// K2/K3: BF16 BRGEMM on tcgen05 tensor cores with the epilogue TPPs fused.
//
// The blocked FC layer (kernels.py:300-329) and the offset-addressed 3x3
// convolution are both a batch-reduce GEMM
//     C[token, feat] = sum_i A_i[token, :] . W_i[feat, :]
// over a sequence of 64-wide reduce blocks i (the reference's k_b channel
// blocks; for the conv the (r, s, c_b) taps).  One persistent CTA per SM
// walks output tiles of 128 tokens x BN features:
//
//   warp 0  TMA producer: per reduce block, one 5-D TMA box of activations
//           (128 x 64 bf16) and one of packed weights (BN x 64 bf16) into a
//           STAGES-deep shared-memory ring (128B swizzle, mbarrier complete_tx)
//   warp 1  MMA issuer: 4 x tcgen05.mma (M=128, N=BN, K=16) per stage into a
//           TMEM accumulator; tcgen05.commit frees the stage / signals the tile
//   warp 2  TMEM allocator (2 x BN columns: the accumulator is double
//           buffered so the epilogue of tile t overlaps the MMAs of tile t+1)
//   warps 4-7  epilogue: tcgen05.ld rows of the accumulator, apply
//           + bias (ops.py:747-782, COL broadcast), ReLU + bitmask / GELU
//           (ops.py:361-366, approx.py:267-276), + residual, RNE narrowing
//           (dtypes.py:82-97) — every op a separately rounded FP32 op in the
//           reference's order — and store to the blocked output layout.
//
// The batch-reduce loop accumulates on chip: C is written exactly once.

#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "sm100.cuh"

// Phase stamps and the TPP_DBG_MODE experiments are compiled in only for
// diagnostic builds (TPP_PHASE_STAMPS=1 at build time): in the product build
// they cost parameter loads and branches on the epilogue's critical path.
#ifdef TPP_PHASE_STAMPS
#define TPP_STAMP(cond, idx, val) \
  do {                            \
    if (p.dbg && (cond)) p.dbg[idx] = (val); \
  } while (0)
#define TPP_DBG_MODE (p.dbg_mode)
#else
#define TPP_STAMP(cond, idx, val) \
  do {                            \
  } while (0)
#define TPP_DBG_MODE 0
#endif

namespace tpp {

using namespace sm100;

namespace tc {

constexpr int BM = 128;          // tokens per tile (UMMA M, TMEM lanes)
constexpr int BK = 64;           // bf16 per reduce block = one 128B swizzle row
// Experiment switch (-DTPP_EPI_GROUPS=3|4 via TPP_NVCC_EXTRA): more epilogue
// warps.  The staging for TMA stores then no longer fits beside the operand
// ring of the big tiles (STG_BUFS = 0), so such builds run with
// TPP_NO_TMA_STORE=1.  Measured on the cfg-5 K=1024 GEMMs (DESIGN 4c): 3
// groups no faster, 4 groups 20 % slower; the product build uses 2.
#ifndef TPP_EPI_GROUPS
#define TPP_EPI_GROUPS 2
#endif
constexpr int kEpiGroups = TPP_EPI_GROUPS;  // epilogue warps per TMEM lane quarter (split the columns)
constexpr int kEpiWarps = 4 * kEpiGroups;
constexpr int kEpiWarp0 = 4;
constexpr int kThreads = 32 * (kEpiWarp0 + kEpiWarps);

enum FeedMode { FEED_FC = 0, FEED_CONV = 1 };

// One operand's walk through a 5-D tensor map.  Tile t starts at element
// t0 = t * rows_per_tile along the tiled axis, split as (t0 % extent) on
// dimension lo_dim and (t0 / extent) on hi_dim.  Each pipeline stage (KPS
// reduce blocks, ONE TMA box) then advances the reduce coordinate:
//   step 0: c[1] += inc, wrapping at `wrap` with a carry into c[3]
//   step 1: c[4] += inc          step 2: c[3] += inc
struct OpFeed {
  int lo_dim, hi_dim, extent, rows_per_tile;
  int step, inc, wrap;
  int sub_bytes;   // smem distance between consecutive reduce blocks of a stage
  int lbo;         // MN-major: distance between 64-wide M/N atoms
};

struct Params {
  int mode;
  int tokens;          // valid rows of the output (M extent)
  int kblocks;         // reduce blocks per tile (multiple of KPS)
  OpFeed fa, fb;       // FC-mode feeds
  int a_mn, b_mn;      // operand major-ness (0 K-major, 1 MN-major)
  // conv: A 5-D map {64, W, H, C_b, N}; 2 output rows x 64 columns per tile
  int cv_P, cv_Q, cv_R, cv_S, cv_pad, cv_Cb, cv_tiles_per_img;
  // ---- tiles ----
  int tiles_m, tiles_n, feats, bn_tile;
  // ---- output / epilogue: out[n_b][m_b][bn][bm] ----
  int o_bn, o_bm, o_mb;
  int act, flags;
  const void* bias;
  const uint16_t* residual;
  void* out;
  uint8_t* mask;        // ReLU bitmask written (TPP_FC_RELU_MASK)
  const uint8_t* mask_in;  // ReLU bitmask applied (RELU_INV, backward-data)
  unsigned long long* dbg;  // optional phase timestamps (CTA 0), tools only
  int dbg_tile;
  int dbg_mode;  // experiments: bit0 skip epilogue math, bit1 skip MMAs
  int tma_store;            // BF16 output through smem staging + TMA (map_c)
  int cv_rows;              // conv: output rows per tile (2, or 4 for RES = 3)
  int cv_wq;                // conv strips (RES = 4): position-space row stride W + pad
  int stage_tx;             // conv strips: bytes one halo box lands (HR x Wq x 128)
  uint16_t* sgd_lo;         // TPP_FC_SGD: lo halves of the split FP32 master (out = hi halves)
  float sgd_lr;
  // stream-K tail (FC mode): work items [0, sk_dp) are whole tiles handed out
  // round-robin; the remaining items' stages (sk_stages in total) are split
  // evenly over the workers.  A tile cut between workers is finished by the
  // worker holding its first stage, which adds the other workers' FP32
  // partials (sk_ws slots, sk_flag handshake) in k order before the epilogue.
  int sk_dp, sk_stages;
  float* sk_ws;
  unsigned* sk_flag;
  // dynamic tile scheduling (FC mode): {ticket, done} counters, zero at
  // launch and reset by the last worker; null = static round-robin
  unsigned* dyn;
  int sleep_waits;   // producer / epilogue waits with a suspend-time hint (experiments: TPP_SLEEP_WAITS)
};

// Dynamic tile queue: the (pair) leader's producer draws work items from a
// global ticket counter and publishes each to its CTA's (and the peer's)
// consumers through a kTQ-deep smem ring (tile id + a full mbarrier per
// slot).  Workers that start late -- e.g. behind a concurrent kernel on
// another stream -- simply draw fewer tiles, so two GEMMs launched side by
// side fill each other's wave-quantisation tails.  The ring needs no empty
// barriers: the producer publishes item k + 1 when it starts loading item k,
// it is at most STAGES items ahead of the MMA, which is at most NBUF items
// ahead of the slowest epilogue warp (TMEM buffers), so a slot is rewritten
// only after every consumer has read it when kTQ > STAGES + NBUF + 2.
constexpr int kTQ = 32;

// One worker's walk over its segments: (work item, first stage, end stage)
struct Seg {
  int tile, k0, k1;
};
struct SegWalk {
  int w, P, dp, S, i, pos, end;
  __device__ __forceinline__ static int sk_begin(const Params& p, int w, int P) {
    return (int)(((long long)w * p.sk_stages) / P);
  }
  __device__ __forceinline__ void start(const Params& p, int w_, int P_, int S_) {
    w = w_; P = P_; S = S_; dp = p.sk_dp; i = 0;
    pos = p.sk_stages ? sk_begin(p, w, P) : 0;
    end = p.sk_stages ? sk_begin(p, w + 1, P) : 0;
  }
  __device__ __forceinline__ bool next(Seg& sg) {
    const int u = w + i * P;
    if (u < dp) {
      sg.tile = u; sg.k0 = 0; sg.k1 = S;
      ++i;
      return true;
    }
    if (pos >= end) return false;
    const int tr = pos / S;
    sg.tile = dp + tr;
    sg.k0 = pos - tr * S;
    sg.k1 = min(S, end - tr * S);
    pos = tr * S + sg.k1;
    return true;
  }
};

// RES = 1: the B operand (conv weights, J = R*S*C_b tap blocks of BN x 64)
// stays resident in smem for the whole kernel; stages then carry only A.
// RES = 2 (conv, halo): additionally each stage is ONE input halo of
// kHaloRows input rows x 64 pixels (all R*S taps of one channel block read
// it through row-shifted descriptors), instead of one A box per tap.
constexpr int kResMaxBytes = 72 * 1024;
constexpr int kHaloRows = 4;   // 2 output rows + R - 1 (R <= 3)
// RES = 3: halo tiles of 4 output rows (two M = 128 accumulators sharing each
// weight tap, 6 halo rows per stage): per output row 1.5 halo rows cross L2->smem
// instead of 2, and the per-tile handoff (commit, accumulator wait, stage wait)
// is paid once per 4 rows
// RES = 4 (conv strips): output positions p = oy * Wq + ox with Wq = W + pad
// -- the right pad of input row y is the left pad of row y + 1, so the halo
// is ONE TMA box of rows Wq pixels wide (x from -pad, OOB zero fill) and tap
// (r, s) of position p reads halo row p + r * Wq + s: a uniform shift across
// row boundaries.  A tile is 256 consecutive positions (two M = 128
// accumulators) regardless of row ends, so only the pad column per row
// (1/57 at W = 56) is wasted instead of 64 - W columns of a 64-wide row, and
// the epilogue stores straight from registers (no smem staging on the port
// the MMAs read operands through).
template <int RES> struct ConvTile {
  static constexpr bool HALO = RES >= 2;
  static constexpr bool STRIP = RES == 4;
  static constexpr int ROWS = RES >= 3 ? 4 : 2;  // output rows per tile (RES 3)
  static constexpr int NACC = ROWS / 2;           // M = 128 accumulators per tile
  static constexpr int HROWS = ROWS + 2;          // input rows per halo (R <= 3, RES 2/3)
};
constexpr int kStripHaloBytes = 66 * 1024;  // >= (Wq - 1 + 256 + 2 Wq + 2 + Wq) pixels x 128 B for Wq <= 64

// CG = 2: CTA pair (cluster of 2, tcgen05 cta_group::2).  The pair computes a
// 256 x BN tile: each CTA stages its own 128 rows of A and HALF of the B rows
// (BN/2), the leader issues M=256 MMAs that read both CTAs' smem and write
// each CTA's TMEM.  Per-SM operand traffic (TMA ingest and the tensor core's
// smem reads) drops by a quarter (BN=256: 48 KB -> 32 KB per 64-deep block).
template <int BN, int STAGES, int KPS, int RES = 0, int CG = 1>
struct Smem {
  static constexpr int A_BYTES = ConvTile<RES>::STRIP ? kStripHaloBytes
                                 : ConvTile<RES>::HALO ? ConvTile<RES>::HROWS * 64 * BK * 2 : KPS * BM * BK * 2;
  static constexpr int B_BYTES = RES ? 0 : KPS * (BN / CG) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // TMEM accumulator buffers: as many as fit in the 512 columns (<= 4).  A
  // tile's tcgen05.ld is served behind the MMAs already queued on the tensor
  // pipe, so with only two buffers the MMAs of tile t + 2 wait for an epilogue
  // that itself waited for tile t + 1's MMAs; 4 buffers let them run on.
  static constexpr int NBUF = 512 / (BN * ConvTile<RES>::NACC) >= 4 ? 4 : 2;
  static constexpr int TMEM_COLS = NBUF * BN * ConvTile<RES>::NACC;
  static constexpr int RES_OFF = STAGES * STAGE_BYTES;
  static constexpr int BAR_OFF = RES_OFF + (RES ? kResMaxBytes : 0);
  // barriers: full[S], empty[S], tfull[NBUF], tempty[NBUF], bres; then tmem base +
  // gelu table (float4 x 512: one entry per 9-bit |x| exponent prefix)
  // + tile queue: tqf[kTQ] barriers, then the tmem slot (16 B), ids[kTQ]
  static_assert(kTQ > STAGES + NBUF + 3, "tile queue shallower than the pipeline");
  static constexpr int TAB_OFF = (BAR_OFF + (2 * STAGES + 2 * NBUF + 1 + kTQ) * 8 + 16 + kTQ * 4 + 15) & ~15;
  // the conv (RES = 2) epilogue has no bias / GELU: no table, no bias staging
  static constexpr int BIAS_OFF = TAB_OFF + (RES >= 2 ? 0 : 512 * 16);    // float [2][256]
  // TMA-store staging: 32 rows x 64 B per epilogue warp, double-buffered
  // when the smem budget allows (a chunk's store need not have left the
  // buffer before the next chunk is staged)
  static constexpr int STG_OFF = (BIAS_OFF + (RES >= 2 ? 0 : 2 * 256 * 4) + 1023) & ~1023;
  static constexpr int STG_BUFS = ConvTile<RES>::STRIP ? 0
                                  : STG_OFF + kEpiWarps * 2048 * 2 + 1024 <= 227 * 1024 ? 2
                                  : STG_OFF + kEpiWarps * 2048 + 1024 <= 227 * 1024 ? 1 : 0;
  static constexpr int BYTES = STG_OFF + kEpiWarps * 2048 * STG_BUFS + 1024;
};

// Register-resident (all indexing resolved at compile time: a dynamically
// indexed coordinate array would live in local memory on the issue path).
struct OpIter {
  int c[5];
  int step, inc, wrap;
  __device__ __forceinline__ void start(const OpFeed& f, int tile) {
    const int t0 = tile * f.rows_per_tile;
    const int lo = t0 % f.extent, hi = t0 / f.extent;
#pragma unroll
    for (int d = 0; d < 5; ++d) c[d] = (d == f.lo_dim ? lo : 0) + (d == f.hi_dim ? hi : 0);
    step = f.step; inc = f.inc; wrap = f.wrap;
  }
  __device__ __forceinline__ void next() {
    if (step == 0) {
      c[1] += inc;
      if (c[1] == wrap) { c[1] = 0; ++c[3]; }
    } else if (step == 1) {
      c[4] += inc;
    } else {
      c[3] += inc;
    }
  }
};

// Producer-side iterator over the stages of one tile: coordinates advance by
// counters (no integer division on the issue path — a single issuing thread
// feeds the tensor core, so its loop must stay short).
struct FeedIter {
  OpIter ai, bi;  // conv mode keeps its A coordinates in ai.c as well
  int cb_n, s_n, pad, s;
  int mode;
  __device__ __forceinline__ void start(const Params& p, int tm, int tn) {
    mode = p.mode;
    bi.start(p.fb, tn);
    if (mode == FEED_FC) {
      ai.start(p.fa, tm);
    } else {
      cb_n = p.cv_Cb; s_n = p.cv_S; pad = p.cv_pad;
      const int n = tm / p.cv_tiles_per_img, pr = tm % p.cv_tiles_per_img;
      s = 0;
      // strips: the halo starts at the input row of the tile's first position
      const int y0 = p.cv_wq ? (pr * 2 * BM) / p.cv_wq : p.cv_rows * pr;
      ai.c[0] = 0; ai.c[1] = -pad; ai.c[2] = y0 - pad; ai.c[3] = 0; ai.c[4] = n;
    }
  }
  __device__ __forceinline__ void next() {
    bi.next();
    if (mode == FEED_FC) {
      ai.next();
    } else {
      // reduce block order (r, s, cb): cb fastest
      if (++ai.c[3] == cb_n) {
        ai.c[3] = 0;
        if (++s == s_n) { s = 0; ++ai.c[2]; ai.c[1] = -pad; } else { ++ai.c[1]; }
      }
    }
  }
};

// global token index of accumulator row r of tile tm (or -1 if padding)
__device__ __forceinline__ int row_token(const Params& p, int tm, int r) {
  if (p.mode == FEED_FC) {
    const int t = tm * BM + r;
    return t < p.tokens ? t : -1;
  }
  const int n = tm / p.cv_tiles_per_img;
  const int pr = tm % p.cv_tiles_per_img;
  const int oh = p.cv_rows * pr + (r >> 6), ow = r & 63;  // accumulator 0 (RES 3 stores through TMA only)
  if (oh >= p.cv_P || ow >= p.cv_Q) return -1;
  return (n * p.cv_P + oh) * p.cv_Q + ow;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float4 lds_f4(uint32_t saddr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(saddr));
  return v;
}

// GELU with the table as one float4 {c0,c1,c2,c3} per interval: one
// ld.shared.v4 at tab_s (shared address) + 16 * clamp(exp-code - 244, 0, 15);
// ~18 instructions per element (the epilogue's issue budget).
// The table is indexed by the 9-bit prefix (|x| bits >> 22) directly, the
// reference's clip(prefix - 244, 0, 15) baked into its 512 entries; prefixes
// >= 260 (|x| >= 8, inf, NaN) hold (1, 0, 0, 0) and |x| is clamped to 8 there,
// so the Horner chain yields exactly the reference's saturated h = 1 (and a
// NaN x still gives NaN through 0.5*x).
__device__ __forceinline__ float gelu4(float x, uint32_t tab_s) {
  const uint32_t xb = __float_as_uint(x);
  const float ax = fminf(fabsf(x), kGeluRangeMax);
  const float4 c = lds_f4(tab_s + ((xb & 0x7FC00000u) >> 18));
  float h = __fadd_rn(__fmul_rn(__fadd_rn(__fmul_rn(__fadd_rn(__fmul_rn(c.w, ax), c.z), ax), c.y), ax), c.x);
  h = __uint_as_float((__float_as_uint(h) & 0x7FFFFFFFu) | (xb & 0x80000000u));  // copysign(h, x)
  return __fmul_rn(__fmul_rn(0.5f, x), __fadd_rn(1.0f, h));
}

// MC > 1: a cluster of MC CTAs along N shares each A (activation) tile: the
// CTAs own consecutive column tiles of one row tile, every reduce block's A box
// is loaded once by CTA (block % MC) and TMA-multicast into all MC CTAs, and a
// stage is free only when every CTA of the cluster has consumed it (each MMA
// commit arrives on the stage's empty barrier in all MC CTAs).  Per-SM L2->SM
// bytes of A drop by MC: the single-wave small layers (cfg 2) are bound by
// the per-SM operand feed, not by the tensor pipe.
template <int BN, int STAGES, int KPS, int RES, int CG, int MC>
__global__ void __launch_bounds__(kThreads, 1)
brgemm_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                 const __grid_constant__ CUtensorMap map_b,
                 const __grid_constant__ CUtensorMap map_c, const Params p) {
  using S = Smem<BN, STAGES, KPS, RES, CG>;
  constexpr bool PAIR = CG == 2;
  static_assert(!PAIR || RES == 0, "CTA pairs stream both operands");
  static_assert(MC == 1 || (CG == 1 && RES == 0), "A multicast: single-CTA MMAs, streamed operands");
  constexpr bool MCAST = MC > 1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128B-swizzled tiles
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + S::NBUF;
  uint64_t* bres = tempty + S::NBUF;
  uint64_t* tqf = bres + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tqf + kTQ);
  int* tq_ids = reinterpret_cast<int*>(tmem_slot + 4);
  float4* gelu_tab = reinterpret_cast<float4*>(smem + S::TAB_OFF);

  TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 0, 0, gtimer());
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // provably warp-uniform: keeps the MMA issuer's descriptor math on the uniform datapath
  const int lane = threadIdx.x & 31;
  // pair mode: work items are 256-row pair tiles, one per cluster; this CTA
  // owns row tile 2*tm + rank and B rows [rank*BN/2, (rank+1)*BN/2) of the tile
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const uint32_t mrank = MCAST ? cluster_ctarank() : 0;
  const int cl_id = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x / MC;
  const int n_cl = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x / MC;
  // work items: pair tiles, multicast groups (MC column tiles of one row tile) or tiles
  const int tiles_ng = p.tiles_n / MC;
  const int num_tiles = (PAIR ? (p.tiles_m + 1) >> 1 : p.tiles_m) * tiles_ng;
  auto tile_mn = [&](int tile, int& tm, int& tn) {
    tm = tile / tiles_ng;
    tn = (tile - tm * tiles_ng) * MC + (int)mrank;
  };
  // stages per tile; halo conv: one per channel block
  using CT = ConvTile<RES>;
  const int nstages = CT::HALO ? p.cv_Cb : p.kblocks / KPS;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
    if (p.tma_store) prefetch_tmap(&map_c);  // the epilogue's first store must not fetch it
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC);
    }
    for (int a = 0; a < S::NBUF; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * CG);
    }
    mbar_init(bres, 1);
    for (int i = 0; i < kTQ; ++i) mbar_init(&tqf[i], 1);
    fence_mbar_init();
  }
  if (warp == 2) {
    if (PAIR) tmem_alloc_pair(tmem_slot, S::TMEM_COLS);
    else tmem_alloc(tmem_slot, S::TMEM_COLS);
  }
  if (!CT::HALO && warp == 3 && p.act == TPP_ACT_GELU) {
    for (int e = lane; e < 512; e += 32) {
      const int j = min(max(e - kGeluBase, 0), 15);
      gelu_tab[e] = e >= kGeluBase + 16
                        ? make_float4(1.0f, 0.0f, 0.0f, 0.0f)
                        : make_float4(__uint_as_float(c_gelu_bits[j]), __uint_as_float(c_gelu_bits[16 + j]),
                                      __uint_as_float(c_gelu_bits[32 + j]), __uint_as_float(c_gelu_bits[48 + j]));
    }
  }
  tc_fence_before();
  if (PAIR || MCAST) cluster_sync();  // the peer signals the leader's barriers / multicast targets ready
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // uniform (MMA operand)
  TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 0, 1, gtimer());
  // Programmatic dependent launch: let the next kernel in the stream be
  // scheduled now (its prologue overlaps our tail).  Each role that touches
  // global memory waits for the previous kernel (griddepcontrol.wait) only
  // after its parameter-derived setup — kernel parameters are immutable, and
  // their first (constant-cache-missing) loads are then off the critical path.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  auto pdl_wait_after = [](int dep) { asm volatile("griddepcontrol.wait;" ::"r"(dep) : "memory"); };

  // ---- dynamic tile queue (p.dyn: FC mode, RES 0, MC 1, no stream-K) ----
  const bool dyn = p.dyn != nullptr;
  const bool q_remote = PAIR && !leader;  // the peer's consumers: slots written by the leader CTA
  // i-th queued work item (-1: none left); one thread per consumer
  auto tq_pop = [&](uint32_t i) -> int {
    const uint32_t slot = i % kTQ, par = (i / kTQ) & 1;
    if (q_remote) mbar_wait_cluster(&tqf[slot], par);
    else mbar_wait(&tqf[slot], par);
    return ld_shared_volatile_s32(smem_u32(&tq_ids[slot]));
  };
  // the leader's producer: publish item i to both CTAs
  auto tq_push = [&](uint32_t i, int t) {
    const uint32_t slot = i % kTQ;
    st_shared_volatile_s32(smem_u32(&tq_ids[slot]), t);
    if (PAIR) {
      st_shared_cluster_s32(mapa_shared(smem_u32(&tq_ids[slot]), 1), t);
      mbar_arrive_cluster(mapa_shared(smem_u32(&tqf[slot]), 1));
    }
    mbar_arrive(&tqf[slot]);
  };
  // items cl_id and cl_id + n_cl are every worker's first two (static: no
  // atomic round trip before the first loads); ticket k is item 2 n_cl + k
  // draw returns the raw ticket; it is converted only where the item is
  // published, a tile later, so the atomic's round trip never stalls the
  // producer (its result register is not touched before then)
  // (inline PTX: atomicAdd() gets warp-aggregated, with a shuffle of the
  // result right behind the atomic -- exactly the stall this avoids)
  auto tq_draw = [&]() -> unsigned {
    unsigned t;
    asm volatile("atom.global.relaxed.gpu.inc.u32 %0, [%1], 0x7fffffff;" : "=r"(t) : "l"(p.dyn) : "memory");  // +1 (tickets stay far below the wrap bound)
    return t;
  };
  auto tq_item = [&](unsigned ticket) -> int {
    const unsigned t = ticket + 2u * (unsigned)n_cl;
    return t < (unsigned)num_tiles ? (int)t : -1;
  };
  // every worker draws exactly one ticket past the end; the last one to
  // finish resets the counters for the next launch on this slot (stream order
  // -- and griddepcontrol.wait before the first draw -- separates the launches)
  auto tq_done = [&] {
    __threadfence();
    if (atomicAdd(p.dyn + 1, 1u) == (unsigned)n_cl - 1) {
      atomicExch(p.dyn, 0u);
      atomicExch(p.dyn + 1, 0u);
    }
  };
  // a warp's work items: lane 0 pops, the id is broadcast.  Dynamic: the
  // following item is popped in the middle of the current one (warp_ahead),
  // so the tile boundary costs a register move, not a barrier round trip
  // (item k + 1 is published when the producer starts item k: never waits)
  auto warp_pop = [&](uint32_t& qi) -> int {
    int t = 0;
    if (lane == 0) t = tq_pop(qi++);
    return __shfl_sync(0xffffffffu, t, 0);
  };
  auto warp_next = [&](SegWalk& w, uint32_t& qi, int& ahead, Seg& sg) -> bool {
    if (!dyn) return w.next(sg);
    const int t = ahead == -2 ? warp_pop(qi) : ahead;  // -2: nothing popped ahead
    ahead = -2;
    sg.tile = t; sg.k0 = 0; sg.k1 = nstages;
    return t >= 0;
  };
  auto warp_ahead = [&](uint32_t& qi, int& ahead, int cur) {
    if (dyn && ahead == -2 && cur >= 0) ahead = warp_pop(qi);
  };

  if (warp == 0 || (RES == 1 && warp == 3)) {
    // ===================== TMA producer(s) =====================
    // RES kernels run two issuing threads (warps 0 and 3) on alternate
    // stages: one thread's TMA issue rate cannot keep up with 128-cycle MMAs.
    constexpr int NPROD = RES == 1 ? 2 : 1;
    const int pid = warp == 0 ? 0 : 1;
    if (lane == 0) {
      FeedIter f;
      SegWalk walk;
      walk.start(p, cl_id, n_cl, nstages);
      Seg sg;
      // dynamic (leader): item k + 1 is published when item k starts and
      // the ticket of item k + 2 drawn then, so neither the peer's producer
      // nor the atomic's round trip ever waits at a tile boundary
      uint32_t qi = 0;
      int nxt = -1;
      unsigned tk = 0;
      bool ended = false;
      auto next_seg = [&](Seg& g) -> bool {
        if (!dyn) return walk.next(g);
        int t;
        if (!q_remote) {
          t = nxt;
          if (t >= 0 && !ended) {
            const int item = tq_item(tk);
            tq_push(qi++, item);
            nxt = item;
            if (item < 0) {
              ended = true;  // tq_done() after the last loads are issued (its fence would stall them)
            } else {
              tk = tq_draw();
            }
          }
        } else {
          t = tq_pop(qi++);
        }
        g.tile = t; g.k0 = 0; g.k1 = nstages;
        return t >= 0;
      };
      bool have;
      if (!dyn || !q_remote) {
        if (dyn) {  // the two static first items, published before the wait
          const int a0 = cl_id < num_tiles ? cl_id : -1;
          const int a1 = a0 >= 0 && cl_id + n_cl < num_tiles ? cl_id + n_cl : -1;
          tq_push(qi++, a0);
          if (a0 >= 0) tq_push(qi++, a1);
          nxt = a1;
          sg.tile = a0; sg.k0 = 0; sg.k1 = nstages;
          have = a0 >= 0;
        } else {
          have = walk.next(sg);
        }
        if (have) {
          int tm, tn;
          tile_mn(sg.tile, tm, tn);
          if (PAIR) f.start(p, 2 * tm + (int)rank, 2 * tn + (int)rank);
          else f.start(p, tm, tn);
        }
        // dynamic: the ticket counter is reset by the previous launch on this slot
        pdl_wait_after(f.ai.c[0] + f.ai.c[1] + f.ai.c[2] + f.ai.c[3] + f.ai.c[4] + f.bi.c[0] + f.bi.c[1] + f.bi.c[2] +
                       f.bi.c[3] + f.bi.c[4] + nstages);
        if (dyn) {
          if (nxt >= 0) tk = tq_draw();
          else ended = true;
        }
      } else {
        have = next_seg(sg);  // the peer: the leader's first item
        if (have) {
          int tm, tn;
          tile_mn(sg.tile, tm, tn);
          f.start(p, 2 * tm + (int)rank, 2 * tn + (int)rank);
        }
        pdl_wait_after(f.ai.c[0] + f.bi.c[0] + nstages);
      }
      TPP_STAMP(blockIdx.x == 0 && pid == 0, 10, gtimer());
      if (RES && pid == 0) {
        // resident weights: every tap block once, on the bres barrier
        const int J = p.kblocks;
        mbar_arrive_expect_tx(bres, J * BN * BK * 2);
        OpIter w;
        w.start(p.fb, 0);
        for (int j = 0; j < J; ++j) {
          tma_load_5d(smem + S::RES_OFF + j * BN * BK * 2, &map_b, bres, w.c[0], w.c[1], w.c[2], w.c[3], w.c[4]);
          w.next();
        }
      }
      int s = 0;
      uint32_t ph = 0;
      uint32_t it = 0;
      // pair: completion bytes of both CTAs count on the leader's full[s]
      const uint32_t full_cl = PAIR ? mapa_shared(smem_u32(full), 0) : 0;
      bool first = true;
      for (; have; have = next_seg(sg), first = false) {
        if (!first) {  // the first segment's feed was set up before the wait
          int tm, tn;
          tile_mn(sg.tile, tm, tn);
          if (PAIR) f.start(p, 2 * tm + (int)rank, 2 * tn + (int)rank);
          else f.start(p, tm, tn);
        }
        for (int j = 0; j < sg.k0; ++j) f.next();  // stream-K: a segment may start mid-tile
        for (int j = sg.k0; j < sg.k1; ++j, ++it) {
          if (NPROD == 1 || (int)(it % NPROD) == pid) {
            if (p.sleep_waits) mbar_wait_sleep(&empty[s], ph ^ 1);
            else mbar_wait(&empty[s], ph ^ 1);
            uint8_t* sa = smem + s * S::STAGE_BYTES;
            if (PAIR) {
              if (leader) mbar_arrive_expect_tx(&full[s], 2 * S::STAGE_BYTES);
              tma_load_5d_pair(sa, &map_a, full_cl + 8 * s, f.ai.c[0], f.ai.c[1], f.ai.c[2], f.ai.c[3], f.ai.c[4]);
              tma_load_5d_pair(sa + S::A_BYTES, &map_b, full_cl + 8 * s, f.bi.c[0], f.bi.c[1], f.bi.c[2], f.bi.c[3],
                               f.bi.c[4]);
            } else if ((TPP_DBG_MODE & 4) && it >= STAGES) {
              mbar_arrive(&full[s]);  // diagnostics: reuse the resident stage, no TMA traffic
            } else {
              mbar_arrive_expect_tx(&full[s], CT::STRIP ? (uint32_t)p.stage_tx : (uint32_t)S::STAGE_BYTES);
              // halo conv: the input box at (cb = j) covering all taps
              if (!MCAST)
                tma_load_5d(sa, &map_a, &full[s], f.ai.c[0], f.ai.c[1], f.ai.c[2], CT::HALO ? j : f.ai.c[3], f.ai.c[4]);
              else if (j % MC == (int)mrank)  // this CTA's share of the cluster's A boxes
                tma_load_5d_mc(sa, &map_a, &full[s], (uint16_t)((1u << MC) - 1), f.ai.c[0], f.ai.c[1], f.ai.c[2],
                               f.ai.c[3], f.ai.c[4]);
              TPP_STAMP(blockIdx.x == 0 && it == 0, 11, gtimer());
              TPP_STAMP(blockIdx.x == 0 && j == 0 && it / nstages < 32, 200 + it / nstages, gtimer());
              if (!RES)
                tma_load_5d(sa + S::A_BYTES, &map_b, &full[s], f.bi.c[0], f.bi.c[1], f.bi.c[2], f.bi.c[3], f.bi.c[4]);
            }
          }
          if (!CT::HALO) f.next();
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
      if (dyn && !q_remote) tq_done();
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread; pair: the leader's) =====================
    if (leader) {  // the whole warp runs the loop (uniform descriptors); one lane issues
      const uint32_t idesc = idesc_bf16_f32(BM * CG, BN, p.a_mn, p.b_mn);
      // K-major: a 16-element K step is +32 B; MN-major: +2 K-groups (+2048 B)
      const uint64_t adesc0 = p.a_mn ? sw128_mnmajor_desc(smem_u32(smem), p.fa.lbo) : sw128_kmajor_desc(smem_u32(smem));
      const uint64_t bdesc0 = (p.b_mn ? sw128_mnmajor_desc(smem_u32(smem), p.fb.lbo) : sw128_kmajor_desc(smem_u32(smem))) +
                              (uint64_t)(S::A_BYTES >> 4);
      const uint32_t astep = p.a_mn ? (2048 >> 4) : (32 >> 4);
      const uint32_t bstep = p.b_mn ? (2048 >> 4) : (32 >> 4);
      const uint32_t asub = (uint32_t)p.fa.sub_bytes >> 4, bsub = (uint32_t)p.fb.sub_bytes >> 4;
      // resident B: tap block j at RES_OFF + j * BN*128 (relative to bdesc0's A_BYTES = 0 base)
      const uint64_t bres0 = sw128_kmajor_desc(smem_u32(smem + S::RES_OFF));
      if (RES) mbar_wait(bres, 0);
      int s = 0;
      uint32_t ph = 0, tcount = 0;
      SegWalk walk;
      walk.start(p, cl_id, n_cl, nstages);
      Seg sg;
      uint32_t qi = 0;
      int ahead = -2;
      for (; warp_next(walk, qi, ahead, sg); ++tcount) {
        const int j0 = sg.k0;
        const uint32_t as = tcount % S::NBUF, aph = (tcount / S::NBUF) & 1;
        mbar_wait(&tempty[as], aph ^ 1);
        TPP_STAMP(blockIdx.x == 0 && lane == 0 && tcount < 32, 240 + tcount, gtimer());
        TPP_STAMP(blockIdx.x == 0 && lane == 0 && (tcount == 4 || tcount == 30), 320 + (tcount == 30) * 2, clock64());
        TPP_STAMP(blockIdx.x == 0 && lane == 0 && (tcount == 4 || tcount == 30), 321 + (tcount == 30) * 2, gtimer());
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + as * (BN * CT::NACC);
        uint64_t strip_off = 0;  // strips: halo row of the tile's first position, 16-byte units
        if (CT::STRIP) {
          const int p0 = (sg.tile % p.cv_tiles_per_img) * 2 * BM;
          strip_off = (uint64_t)((p0 - (p0 / p.cv_wq) * p.cv_wq) * 8);
        }
        for (int j = j0; j < sg.k1; ++j) {
          mbar_wait(&full[s], ph);
          TPP_STAMP(blockIdx.x == 0 && lane == 0 && tcount == p.dbg_tile && j == 0, 2, gtimer());
          TPP_STAMP(blockIdx.x == 0 && lane == 0 && tcount < 32 && j == 0, 16 + 4 * tcount, gtimer());
          tc_fence_after();
          // descriptor start-address field is in 16-byte units
          const uint64_t soff = (uint64_t)((s * S::STAGE_BYTES) >> 4);
          if (CT::HALO) {
            // tap (r, s) of channel block j: A rows start at halo row r*64 + s
            // (the 128B swizzle is address-based, so a row-shifted start is a
            // valid K-major view); weights block (r*S + s)*C_b + j is resident
            const uint64_t a0 = adesc0 + soff;
            const uint64_t b0 = bres0 + (uint64_t)((j * BN * BK * 2) >> 4);
            const uint64_t btap = (uint64_t)((p.cv_Cb * BN * BK * 2) >> 4);
            if (CT::STRIP) {
              // tap (r, s), accumulator h: halo row off + h * 128 + r * Wq + s
              const uint64_t a1 = a0 + strip_off;
              const uint64_t wq8 = (uint64_t)p.cv_wq * 8;
#pragma unroll
              for (int tap = 0; tap < 9; ++tap) {
                const uint64_t bd = b0 + btap * tap;
                const uint64_t at = a1 + wq8 * (tap / 3) + 8 * (tap % 3);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                  for (int kk = 0; kk < BK / 16; ++kk)
                    umma_f16_warp(tmem_d + h * BN, at + (uint64_t)(h * BM * 8) + 2 * kk, bd + 2 * kk, idesc,
                                  (j > j0 || tap > 0 || kk > 0) ? 1u : 0u);
                }
              }
            } else if (p.cv_R == 3 && p.cv_S == 3) {
              // 3x3: every descriptor offset is an immediate (the single
              // issuing thread must keep pace with 48-cycle N=64 MMAs)
#pragma unroll
              for (int tap = 0; tap < 9; ++tap) {
                const uint64_t bd = b0 + btap * tap;
#pragma unroll
                for (int h = 0; h < CT::NACC; ++h) {  // accumulator h: output rows 2h, 2h + 1 of the tile
                  const uint64_t ad = a0 + (uint64_t)(((((tap / 3) + 2 * h) * 64 + tap % 3) * 128) >> 4);
#pragma unroll
                  for (int kk = 0; kk < BK / 16; ++kk)
                    if (!(TPP_DBG_MODE & 2))
                      umma_f16_warp(tmem_d + h * BN, ad + 2 * kk, bd + 2 * kk, idesc,
                                    (j > j0 || tap > 0 || kk > 0) ? 1u : 0u);
                }
              }
            } else {
              for (int rr = 0; rr < p.cv_R; ++rr) {
                for (int ss = 0; ss < p.cv_S; ++ss) {
                  const uint64_t bd = b0 + btap * (rr * p.cv_S + ss);
#pragma unroll
                  for (int h = 0; h < CT::NACC; ++h) {
                    const uint64_t ad = a0 + (uint64_t)((((rr + 2 * h) * 64 + ss) * 128) >> 4);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)
                      umma_f16_warp(tmem_d + h * BN, ad + 2 * kk, bd + 2 * kk, idesc,
                                    (j > j0 || rr > 0 || ss > 0 || kk > 0) ? 1u : 0u);
                  }
                }
              }
            }
          } else {
#pragma unroll
            for (int kb = 0; kb < KPS; ++kb) {
              const uint64_t bd = RES ? bres0 + (uint64_t)((j * BN * BK * 2) >> 4) : bdesc0 + soff + bsub * kb;
#pragma unroll
              for (int kk = 0; kk < BK / 16; ++kk) {
                if (TPP_DBG_MODE & 2) continue;
                if (PAIR)
                  umma_f16_pair_warp(tmem_d, adesc0 + soff + asub * kb + astep * kk, bd + bstep * kk, idesc,
                                (j > j0 || kb > 0 || kk > 0) ? 1u : 0u);
                else
                  umma_f16_warp(tmem_d, adesc0 + soff + asub * kb + astep * kk, bd + bstep * kk,
                           idesc, (j > j0 || kb > 0 || kk > 0) ? 1u : 0u);
              }
            }
          }
          if (PAIR) umma_commit_pair_warp(&empty[s], 3);
          else if (MCAST) umma_commit_mc_warp(&empty[s], (uint16_t)((1u << MC) - 1));
          else umma_commit_warp(&empty[s]);
          if (++s == STAGES) { s = 0; ph ^= 1; }
          warp_ahead(qi, ahead, sg.tile);  // the MMAs of this stage are queued: slack
        }
        if (PAIR) umma_commit_pair_warp(&tfull[as], 3);
        else umma_commit_warp(&tfull[as]);
        TPP_STAMP(blockIdx.x == 0 && lane == 0 && tcount == p.dbg_tile, 3, gtimer());
        TPP_STAMP(blockIdx.x == 0 && lane == 0 && tcount < 32, 17 + 4 * tcount, gtimer());
      }
    }
  } else if (warp >= kEpiWarp0) {
    // ===================== epilogue (8 warps) =====================
    pdl_wait_after(p.flags ^ p.tiles_n ^ p.feats ^ p.o_bn ^ p.o_bm ^ p.o_mb ^ p.act ^ p.tma_store ^ p.mode ^ p.tokens);
    const int ew = warp - kEpiWarp0;
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int grp = ew >> 2;           // 32-column chunks grp, grp + kEpiGroups, ...
    const int r = q * 32 + lane;
    float* bias_s = reinterpret_cast<float*>(smem + S::BIAS_OFF);
    uint8_t* stg0 = smem + S::STG_OFF + ew * 2048 * S::STG_BUFS;  // 32 rows x 64 B, 64B-swizzled
    uint32_t nstore = 0;
    uint32_t tcount = 0;
    SegWalk walk;
    walk.start(p, cl_id, n_cl, nstages);
    Seg sg;
    uint32_t qi = 0;
    int ahead = -2;
    for (; warp_next(walk, qi, ahead, sg); ++tcount) {
      const int tile = sg.tile;
      int tm, tn;
      tile_mn(tile, tm, tn);
      if (PAIR) tm = 2 * tm + (int)rank;
      // partial bookkeeping: `park` stores this segment's FP32 partial in
      // slot park_slot and skips the epilogue; otherwise nsrc parked partials
      // (slots src_base + j * src_step, k order) are added before it
      bool park = false;
      int park_slot = 0, nsrc = 0, src_base = 0, src_step = 1;
      if (p.sk_stages) {  // stream-K tail: the worker with the first stage finishes
        if (sg.k0 > 0) {
          park = true;
          park_slot = cl_id;
        } else if (sg.k1 < nstages) {
          const int tile_end = (tile - p.sk_dp + 1) * nstages;
          int w1 = cl_id + 1;
          while (w1 < n_cl && SegWalk::sk_begin(p, w1, n_cl) < tile_end) ++w1;
          nsrc = w1 - cl_id - 1;
          src_base = cl_id + 1;
        }
      }
      const uint32_t as = tcount % S::NBUF, aph = (tcount / S::NBUF) & 1;
      float* bs = bias_s + (tcount & 1) * 256;
      if (p.flags & TPP_FC_BIAS) {
        // stage this tile's bias (COL broadcast) in smem while the MMAs run
        for (int i = ew * 32 + lane; i < BN; i += kEpiWarps * 32) {
          const int f = tn * BN + i;
          float v = 0.0f;
          if (f < p.feats)
            v = (p.flags & TPP_FC_BIAS_FP32) ? reinterpret_cast<const float*>(p.bias)[f]
                                             : bf16_to_f32(reinterpret_cast<const uint16_t*>(p.bias)[f]);
          bs[i] = v;
        }
        named_bar_sync(1, kEpiWarps * 32);
      }
      // Index arithmetic (integer divisions) is done while the accumulator is
      // still being computed; the empty asm pins it before the wait.
      // token coordinates only for the paths that address rows themselves
      const bool need_rows = !p.tma_store || (p.flags & (TPP_FC_RELU_INV | TPP_FC_RESIDUAL | TPP_FC_OUT_FP32 | TPP_FC_SGD)) ||
                             (p.act == TPP_ACT_RELU && (p.flags & TPP_FC_RELU_MASK));
      int t = 0, nb = 0, n_in = 0;
      if (need_rows) {
        t = row_token(p, tm, r);
        nb = t >= 0 ? t / p.o_bn : 0;
        n_in = t >= 0 ? t % p.o_bn : 0;
      }
      // TMA store box of this warp: 32 rows x 32 features.  FC: 32 consecutive
      // tokens of one token block; conv: 32 pixels of one output row.
      int sc1, sc2, sc4;
      bool warp_rows;
      if (p.mode == FEED_FC) {
        const int t0 = tm * BM + q * 32;
        sc1 = 0; sc2 = t0 % p.o_bn; sc4 = t0 / p.o_bn;
        warp_rows = p.tma_store && t0 < p.tokens;
      } else {
        const int img = tm / p.cv_tiles_per_img;
        sc2 = CT::ROWS * (tm - img * p.cv_tiles_per_img) + (q >> 1);
        sc1 = (q & 1) * 32; sc4 = img;
        warp_rows = p.tma_store && sc2 < p.cv_P && sc1 < p.cv_Q;
      }
      asm volatile("" ::"r"(t), "r"(nb), "r"(n_in), "r"(sc1), "r"(sc2), "r"(sc4), "r"((int)warp_rows));
      if (p.sleep_waits) mbar_wait_sleep(&tfull[as], aph);
      else mbar_wait(&tfull[as], aph);
      warp_ahead(qi, ahead, tile);
      TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128 && tcount == p.dbg_tile, 4, gtimer());
      TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128 && tcount == p.dbg_tile, 189, clock64());
      TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128 && tcount < 32, 18 + 4 * tcount, gtimer());
      tc_fence_after();
      // chunk c: accumulator c / nch1, 32 columns (grp + (c % nch1) * kEpiGroups) * 32
      const int nch1 = (BN / 32 - grp + kEpiGroups - 1) / kEpiGroups;
      const int nch = nch1 * CT::NACC;
      const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + as * (BN * CT::NACC);
      auto chunk_col = [&](int c) { return (grp + (CT::NACC > 1 ? c % nch1 : c) * kEpiGroups) * 32; };
      auto chunk_acc = [&](int c) { return CT::NACC > 1 ? c / nch1 : 0; };
      uint32_t v[32];
      if (nch > 0) tmem_ld32(tacc + grp * 32, v);
      TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128 && tcount == p.dbg_tile, 188, clock64());
      // release this warp's share of the accumulator as soon as its last
      // chunk is in registers, so the next tile's MMAs can start while the
      // math and stores of this one proceed
      TPP_STAMP(blockIdx.x == 0 && lane == 0 && tcount == 20, 300 + ew, gtimer());
      auto release = [&] {
        TPP_STAMP(blockIdx.x == 0 && lane == 0 && tcount == 20, 280 + ew, gtimer());
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR && !leader) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[as]), 0));
          else mbar_arrive(&tempty[as]);
        }
      };
      if (nch <= 0) release();
      if (nsrc > 0) {  // the parked partials of this tile must have landed
        if (lane == 0)
          for (int j = 0; j < nsrc; ++j) {
            const unsigned* fl = p.sk_flag + (src_base + j * src_step) * CG + (int)rank;
            unsigned v;
            do {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl) : "memory");
            } while (v == 0);
          }
        __syncwarp();
      }
#pragma unroll 1
      for (int ch = 0; ch < nch; ++ch) {
        const int col = chunk_col(ch);
        const int hacc = chunk_acc(ch);
        tmem_ld_wait();
        float x[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(v[i]);
        // the next chunk's TMEM load overlaps this chunk's math and stores
        if (ch + 1 < nch) tmem_ld32(tacc + chunk_acc(ch + 1) * BN + chunk_col(ch + 1), v);
        else release();
        if (park) {  // park this segment's FP32 partial (slot [128 rows][BN])
          // slot layout [BN/4][128 rows][4]: a warp's 32 rows of one column quad
          // are 512 contiguous bytes (coalesced stores and loads)
          float4* dst = reinterpret_cast<float4*>(p.sk_ws + (size_t)(park_slot * CG + (int)rank) * BM * BN) +
                        (col / 4) * BM + r;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            __stcg(dst + i * BM, make_float4(x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3]));
          continue;
        }
        for (int j = 0; j < nsrc; ++j) {  // the other k ranges, in slot order
          const float4* src =
              reinterpret_cast<const float4*>(p.sk_ws + (size_t)((src_base + j * src_step) * CG + (int)rank) * BM * BN) +
              (col / 4) * BM + r;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 q4 = __ldcg(src + i * BM);
            x[4 * i] = __fadd_rn(x[4 * i], q4.x); x[4 * i + 1] = __fadd_rn(x[4 * i + 1], q4.y);
            x[4 * i + 2] = __fadd_rn(x[4 * i + 2], q4.z); x[4 * i + 3] = __fadd_rn(x[4 * i + 3], q4.w);
          }
        }
        TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128 && tcount == p.dbg_tile && ch == 0, 7, gtimer());
        TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128 && tcount == p.dbg_tile && ch < 8, 150 + 4 * ch + 0, clock64());
        if (CT::STRIP) {
          // position p0 + hacc * 128 + r of image n -> output pixel (oy, ox);
          // the pad column (ox >= Q) and positions past the image are dropped
          const int img = tm / p.cv_tiles_per_img;
          const int pos = (tm - img * p.cv_tiles_per_img) * 2 * BM + hacc * BM + r;
          const int oy = pos / p.cv_wq, ox = pos - oy * p.cv_wq;
          if (ox < p.cv_Q && oy < p.cv_P) {
            uint32_t w[16];
            pack_bf16_ref_n<16>(x, w);
            // two 256-bit stores: full 32-byte sectors (a warp's 32 positions
            // are 32 different lines; 16-byte pieces cost twice the L1 wavefronts)
            uint16_t* op = reinterpret_cast<uint16_t*>(p.out) +
                           ((((int64_t)img * p.o_mb + tn) * p.cv_P + oy) * p.cv_Q + ox) * 64 + col;
            st_global_v8(op, w);
            st_global_v8(op + 16, w + 8);
          }
          continue;
        }
        const int f0 = tn * BN + col;
        if (TPP_DBG_MODE & 1) continue;
        if (f0 >= p.feats || (!p.tma_store && t < 0)) continue;
        const int mb = p.o_bm == 64 ? f0 >> 6 : f0 / p.o_bm, m_in = f0 - mb * p.o_bm;
        const int64_t row_off = ((int64_t)(nb * p.o_mb + mb) * p.o_bn + n_in);
        if (p.flags & TPP_FC_BIAS) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 b4 = lds_f4(smem_u32(bs + col + i));
            x[i] = __fadd_rn(x[i], b4.x); x[i + 1] = __fadd_rn(x[i + 1], b4.y);
            x[i + 2] = __fadd_rn(x[i + 2], b4.z); x[i + 3] = __fadd_rn(x[i + 3], b4.w);
          }
        }
        if ((p.flags & TPP_FC_RELU_INV) && t >= 0) {
          // ops.py:367-369: where(mask, dy, 0) with the forward ReLU bitmask
          const uint32_t bits = *reinterpret_cast<const uint32_t*>(p.mask_in + row_off * (p.o_bm / 8) + m_in / 8);
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = ((bits >> i) & 1u) ? x[i] : 0.0f;
        }
        if (p.act == TPP_ACT_RELU) {
          if ((p.flags & TPP_FC_RELU_MASK) && t >= 0) {
            uint32_t bits = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) bits |= (x[i] > 0.0f ? 1u : 0u) << i;
            *reinterpret_cast<uint32_t*>(p.mask + row_off * (p.o_bm / 8) + m_in / 8) = bits;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = relu_f(x[i]);
        } else if (p.act == TPP_ACT_GELU) {
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = gelu4(x[i], smem_u32(gelu_tab));
        }
        TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128 && tcount == p.dbg_tile && ch < 8, 150 + 4 * ch + 1, clock64());
        if ((p.flags & TPP_FC_RESIDUAL) && t >= 0) {
          const uint4* rp = reinterpret_cast<const uint4*>(p.residual + row_off * p.o_bm + m_in);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint4 r4 = __ldg(rp + i);
            const uint32_t w[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              x[8 * i + 2 * e] = __fadd_rn(x[8 * i + 2 * e], __uint_as_float(w[e] << 16));
              x[8 * i + 2 * e + 1] = __fadd_rn(x[8 * i + 2 * e + 1], __uint_as_float(w[e] & 0xFFFF0000u));
            }
          }
        }
        if (p.flags & TPP_FC_SGD) {
          // split-SGD on the FP32 master, in place (kernels.py:235-251; the
          // split_sgd_vec_kernel arithmetic): w = hi:lo, w - g*lr, re-split
          uint4* hp = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.out) + row_off * p.o_bm + m_in);
          uint4* lp = reinterpret_cast<uint4*>(p.sgd_lo + row_off * p.o_bm + m_in);
          uint4 hv[4], lv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            hv[i] = hp[i];
            lv[i] = lp[i];
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t hw[4] = {hv[i].x, hv[i].y, hv[i].z, hv[i].w}, lw[4] = {lv[i].x, lv[i].y, lv[i].z, lv[i].w};
            uint32_t oh[4], ol[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float w0 = __uint_as_float((hw[q] << 16) | (lw[q] & 0xFFFFu));
              const float w1 = __uint_as_float((hw[q] & 0xFFFF0000u) | (lw[q] >> 16));
              const uint32_t r0 = __float_as_uint(__fsub_rn(w0, __fmul_rn(x[8 * i + 2 * q], p.sgd_lr)));
              const uint32_t r1 = __float_as_uint(__fsub_rn(w1, __fmul_rn(x[8 * i + 2 * q + 1], p.sgd_lr)));
              oh[q] = (r0 >> 16) | (r1 & 0xFFFF0000u);
              ol[q] = (r0 & 0xFFFFu) | (r1 << 16);
            }
            hp[i] = make_uint4(oh[0], oh[1], oh[2], oh[3]);
            lp[i] = make_uint4(ol[0], ol[1], ol[2], ol[3]);
          }
        } else if (p.flags & TPP_FC_OUT_FP32) {
          float4* op = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + row_off * p.o_bm + m_in);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            op[i] = make_float4(x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3]);
        } else if (p.tma_store) {
          uint32_t w[16];
          pack_bf16_ref_n<16>(x, w);
        TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128 && tcount == p.dbg_tile && ch < 8, 150 + 4 * ch + 2, clock64());
          uint4 val[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) val[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
          uint8_t* stg = stg0 + (nstore % S::STG_BUFS) * 2048;
          if (lane == 0) {  // the store that last used this buffer has read it
            if (S::STG_BUFS == 2) bulk_wait_read<1>();
            else bulk_wait_read<0>();
          }
          __syncwarp();
          // row `lane`, 16-byte chunk c lands at chunk c ^ ((lane >> 1) & 3) (SWIZZLE_64B)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            st_shared_v4(smem_u32(stg + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)), val[c]);
          fence_async_smem();
          __syncwarp();
          ++nstore;
          if (lane == 0) {
            // every chunk commits a bulk group (possibly empty) so that the
            // per-buffer wait_group counts stay aligned with nstore
            // RES 3: accumulator h holds output rows 2h, 2h + 1 of the tile
            if (CT::NACC == 1 ? warp_rows : (p.tma_store && sc2 + 2 * hacc < p.cv_P && sc1 < p.cv_Q))
              tma_store_5d(&map_c, stg, m_in, sc1, sc2 + 2 * hacc, mb, sc4);
            bulk_commit();
        TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128 && tcount == p.dbg_tile && ch < 8, 150 + 4 * ch + 3, clock64());
          }
        } else {
          uint16_t* op = reinterpret_cast<uint16_t*>(p.out) + row_off * p.o_bm + m_in;
          uint32_t w[16];
          pack_bf16_ref_n<16>(x, w);
          if ((reinterpret_cast<uintptr_t>(op) & 31) == 0) {  // full 32-byte sectors
            st_global_v8(op, w);
            st_global_v8(op + 16, w + 8);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              reinterpret_cast<uint4*>(op)[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
          }
        }
      }
      if (park || nsrc > 0) {
        // publish the parked partial / recycle the consumed flags (every
        // epilogue thread's stores are fenced before the barrier)
        if (park) __threadfence();
        named_bar_sync(2, kEpiWarps * 32);
        if (ew == 0 && lane == 0) {
          if (park) {
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.sk_flag + park_slot * CG + (int)rank), "r"(1u)
                         : "memory");
          } else {
            for (int j = 0; j < nsrc; ++j) p.sk_flag[(src_base + j * src_step) * CG + (int)rank] = 0u;
          }
        }
      }
      TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128 && tcount == p.dbg_tile, 8, gtimer());
      TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128 && tcount == p.dbg_tile, 5, gtimer());
      TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128 && tcount < 32, 19 + 4 * tcount, gtimer());
      TPP_STAMP(blockIdx.x == 0 && lane == 0 && tcount == 20, 290 + ew, gtimer());
    }
    // smem must outlive the bulk stores' reads; their global writes complete
    // with the grid (what the next kernel's griddepcontrol.wait observes)
    TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128, 190, clock64());
    if (lane == 0 && p.tma_store) bulk_wait_read<0>();
    TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128, 191, clock64());
  }

  tc_fence_before();
  if (PAIR || MCAST) cluster_sync();  // no CTA leaves while the cluster still uses its smem / TMEM / barriers
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (PAIR) tmem_dealloc_pair(tmem_base, S::TMEM_COLS);
    else tmem_dealloc(tmem_base, S::TMEM_COLS);
  }
  TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 64, 6, gtimer());
  TPP_STAMP(blockIdx.x == 0 && threadIdx.x == 128, 192, clock64());
}

// ---------------------------------------------------------------------------
// host side: tensor maps (driver entry point, no -lcuda), launch
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 5-D bf16 map, dims innermost first, strides in bytes for dims 1..4
// Encoded maps are cached per thread (the same layer calls encode the same
// three maps every time; cuTensorMapEncodeTiled costs ~2-3 us of host time
// per map, more than a small layer's kernel): key = every encode argument.
struct MapKey {
  const void* base;
  uint64_t dims[5], strides[4];
  uint32_t box[5];
  int swz, dt;
  bool operator==(const MapKey& o) const { return memcmp(this, &o, sizeof(MapKey)) == 0; }
};
struct MapCache {
  static constexpr int N = 48;
  MapKey key[N];
  CUtensorMap map[N];
  int used = 0, next = 0;
};

static int make_map_5d(CUtensorMap* m, const void* base, const uint64_t dims[5],
                       const uint64_t strides[4], const uint32_t box[5],
                       CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B,
                       CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) {
  thread_local MapCache cache;
  MapKey k;
  memset(&k, 0, sizeof(k));
  k.base = base;
  memcpy(k.dims, dims, sizeof(k.dims));
  memcpy(k.strides, strides, sizeof(k.strides));
  memcpy(k.box, box, sizeof(k.box));
  k.swz = (int)swz;
  k.dt = (int)dt;
  for (int i = 0; i < cache.used; ++i)
    if (cache.key[i] == k) {
      *m = cache.map[i];
      return TPP_OK;
    }
  auto enc = get_encode();
  if (!enc) return fail(TPP_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (reinterpret_cast<uintptr_t>(base) % 16) return fail(TPP_E_TENSOR, "TMA base not 16B aligned");
  cuuint64_t gd[5];
  cuuint64_t gs[4];
  cuuint32_t bd[5], es[5];
  for (int i = 0; i < 5; ++i) {
    gd[i] = dims[i];
    bd[i] = box[i];
    es[i] = 1;
  }
  for (int i = 0; i < 4; ++i) {
    if (strides[i] % 16) return fail(TPP_E_TENSOR, "TMA stride not a multiple of 16 bytes");
    gs[i] = strides[i];
  }
  CUresult r = enc(m, dt, 5, const_cast<void*>(base), gd, gs, bd,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TPP_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  const int slot = cache.used < MapCache::N ? cache.used++ : (cache.next++ % MapCache::N);
  cache.key[slot] = k;
  cache.map[slot] = *m;
  return TPP_OK;
}

// The stream-K tail is OFF by default: measured on the cfg-5 GEMMs it was
// slower than whole tiles (fwd 8192x4096->1024: 78 vs 56 us; dW 4096^2 over
// 8192 tokens: 223 vs 215 us; dW 1024x4096: 86 vs 78 us, tools/sk_probe.py) —
// segments that start mid-K break the lock-step K sweep the concurrent tiles
// share in L2, and the finisher's partial reads sit on the critical path.
// TPP_STREAMK=1 enables it (experiments; tests/test_gpu_dispatch.py checks
// its numerics when set).
static bool env_no_streamk() {
  static const bool v = getenv("TPP_STREAMK") == nullptr;
  return v;
}

// Stream-K partial slots + flags, one buffer per device, allocated on first
// use outside a CUDA-graph capture (inside a capture without it the GEMM runs
// without the stream-K tail).  The flags are reset by their consumers, so the
// buffer is reusable by every later launch; stream-K GEMMs of one device must
// not run concurrently on two streams.
static float* sk_workspace(cudaStream_t stream, size_t floats, unsigned** flags) {
  static std::mutex mu;
  static std::unordered_map<int, std::pair<float*, size_t>> bufs;
  constexpr size_t kFlagBytes = 64 * 1024;   // 16K slot flags
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  auto it = bufs.find(dev);
  if (it == bufs.end() || it->second.second < floats) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
    if (it != bufs.end()) {
      cudaDeviceSynchronize();
      cudaFree(it->second.first);
      bufs.erase(it);
    }
    const size_t want = floats < ((size_t)19 << 20) / 4 ? ((size_t)19 << 20) / 4 : floats;
    void* ptr = nullptr;
    if (cudaMalloc(&ptr, kFlagBytes + want * sizeof(float)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    cudaMemset(ptr, 0, kFlagBytes);
    cudaDeviceSynchronize();
    it = bufs.emplace(dev, std::make_pair(reinterpret_cast<float*>(static_cast<char*>(ptr) + kFlagBytes), want)).first;
  }
  *flags = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(it->second.first) - kFlagBytes);
  return it->second.first;
}

// Dynamic tile scheduling: FC-mode GEMMs flagged TPP_FC_DYNAMIC_TILES (the
// overlapped backward of BlockedMLP), or all of them under
// tpp_set_tile_scheduling(1).  Alone, a GEMM runs as fast either way
// (tools/dyn_ab.py: within 1-3 %); side by side on two streams the dynamic
// draw lets each fill the other's idle SMs.
static std::atomic<int> g_tile_mode{-1};  // -1: not yet read from the environment
static int tile_mode() {
  int v = g_tile_mode.load(std::memory_order_relaxed);
  if (v < 0) {
    int want = getenv("TPP_STATIC_TILES") != nullptr ? 2 : 0, expect = -1;
    g_tile_mode.compare_exchange_strong(expect, want);
    v = g_tile_mode.load(std::memory_order_relaxed);
  }
  return v;
}
}  // namespace tc
int set_tile_scheduling(int mode) {
  const int prev = tc::tile_mode();
  if (mode >= 0 && mode <= 2) tc::g_tile_mode.store(mode);
  return prev;
}
namespace tc {

// Ticket counters for dynamic tile scheduling: one 32-byte slot {ticket, done}
// per (device, stream).  Launches on one stream are ordered (a PDL successor
// draws only after griddepcontrol.wait, i.e. after its predecessor's reset),
// so a slot is never shared by two running kernels; kernels on different
// streams -- the concurrent GEMMs this exists for -- use different slots.  The
// buffer is allocated and zeroed once per device, outside any graph capture
// (a capture before first use runs the static walk).  A captured graph keeps
// its capture streams' slots: it must not be replayed concurrently with other
// work on those streams.
static unsigned* dyn_counter(cudaStream_t stream) {
  constexpr int kSlots = 4096, kStride = 8;
  struct Dev {
    unsigned* buf = nullptr;
    std::unordered_map<cudaStream_t, int> slot;
  };
  static std::mutex mu;
  static std::unordered_map<int, Dev> devs;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  Dev& d = devs[dev];
  if (!d.buf) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return nullptr;
    }
    void* ptr = nullptr;
    if (cudaMalloc(&ptr, (size_t)kSlots * kStride * sizeof(unsigned)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    if (cudaMemset(ptr, 0, (size_t)kSlots * kStride * sizeof(unsigned)) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
      cudaGetLastError();
      cudaFree(ptr);
      return nullptr;
    }
    d.buf = static_cast<unsigned*>(ptr);
  }
  auto it = d.slot.find(stream);
  if (it == d.slot.end()) {
    if ((int)d.slot.size() >= kSlots) return nullptr;
    it = d.slot.emplace(stream, (int)d.slot.size()).first;
  }
  return d.buf + (size_t)it->second * kStride;
}

template <int BN, int STAGES, int KPS, int RES = 0, int CG = 1, int MC = 1>
static int launch_cfg(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                      const Params& p, cudaStream_t stream) {
  using S = Smem<BN, STAGES, KPS, RES, CG>;
  static_assert(S::BYTES <= 227 * 1024, "shared memory budget");
  static_assert(TPP_EPI_GROUPS != 2 || ConvTile<RES>::STRIP || S::STG_BUFS > 0, "product build: TMA-store staging must fit");
  if (S::STG_BUFS == 0 && p.tma_store && !ConvTile<RES>::STRIP)  // experiment builds only
    return fail(TPP_E_UNSUPPORTED, "no TMA-store staging in this build: set TPP_NO_TMA_STORE=1");
  auto kern = brgemm_tc_kernel<BN, STAGES, KPS, RES, CG, MC>;
  constexpr int CL = CG * MC;  // cluster size (one of CG, MC is 1)
  {
    cudaError_t e = ensure_smem_attr((const void*)kern, S::BYTES);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(brgemm_tc_kernel)");
  }
  static int max_clusters = 0;
  static std::once_flag once;
  std::call_once(once, [&] {
    max_clusters = num_sms() / CL;
    if (CL > 1) {
      // co-resident pairs (SM pairs of one TPC) — a persistent grid must not exceed it
      cudaLaunchConfig_t q{};
      q.gridDim = dim3(num_sms());
      q.blockDim = dim3(kThreads);
      q.dynamicSmemBytes = S::BYTES;
      cudaLaunchAttribute ca[1];
      ca[0].id = cudaLaunchAttributeClusterDimension;
      ca[0].val.clusterDim.x = CL; ca[0].val.clusterDim.y = 1; ca[0].val.clusterDim.z = 1;
      q.attrs = ca;
      q.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &q) == cudaSuccess && n > 0 && n < max_clusters) max_clusters = n;
      cudaGetLastError();
    }
  });
  const int units = (CG > 1 ? (p.tiles_m + 1) / 2 : p.tiles_m) * (p.tiles_n / MC);
  int grid = CL * (units < max_clusters ? units : max_clusters);
  Params pk = p;
  pk.sk_dp = units;   // default: every work item whole, round-robin
  pk.sk_stages = 0;
  if (RES == 0 && MC == 1 && p.mode == FEED_FC) {
    const int S = p.kblocks / KPS;
    // (split-K of every tile into 2-4 K parts, part-major, was measured
    // slower on every cfg-5 shape -- the FP32 partial round trip costs more
    // than the idle tail it removes: fwd 8192x4096->1024 92 vs 56 us, dW
    // 4096^2 219 vs 215 us, dW 1024x4096 93 vs 78 us -- and is not built)
    // stream-K tail (opt-in, TPP_STREAMK=1)
    const int workers = grid / CL;
    if (units > workers && units % workers != 0 && (units % workers) * 10 < workers * 9 &&
        S >= 4 && !env_no_streamk()) {
      unsigned* flags = nullptr;
      float* ws = sk_workspace(stream, (size_t)workers * CG * BM * BN, &flags);
      if (ws) {
        pk.sk_dp = (units / workers - 1) * workers;
        pk.sk_stages = (units - pk.sk_dp) * S;
        pk.sk_ws = ws;
        pk.sk_flag = flags;
      }
    }
  }
  static const int sleep_waits = getenv("TPP_SLEEP_WAITS") ? atoi(getenv("TPP_SLEEP_WAITS")) : 0;
  pk.sleep_waits = sleep_waits;
  pk.dyn = nullptr;
  if (RES == 0 && MC == 1 && p.mode == FEED_FC && pk.sk_stages == 0 && units > 1 &&
      (tile_mode() == 1 || (tile_mode() == 0 && (p.flags & TPP_FC_DYNAMIC_TILES))))
    pk.dyn = dyn_counter(stream);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = S::BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_allowed();
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = CL; attr[1].val.clusterDim.y = 1; attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = CL > 1 ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, mc, pk);
  if (e != cudaSuccess) return cuda_status(e, "cudaLaunchKernelEx(brgemm_tc_kernel)");
  TPP_CUDA_LAUNCH_CHECK("brgemm_tc_kernel");
  set_last_config("brgemm_tc_kernel<" + std::to_string(BN) + "," + std::to_string(STAGES) + "," +
                  std::to_string(KPS) + "," + std::to_string(RES) + "," + std::to_string(CG) + "," +
                  std::to_string(MC) + "> grid=" + std::to_string(grid) + " tiles=" + std::to_string(p.tiles_m) +
                  "x" + std::to_string(p.tiles_n) +
                  (pk.sk_stages ? " streamk=" + std::to_string(units - pk.sk_dp) + "/" + std::to_string(units)
                                : std::string()) +
                  (pk.dyn ? " dyn" : ""));
  return TPP_OK;
}

// (tile width, reduce blocks per stage, CTAs per MMA) -> instantiation; stages fill ~192 KB
static int launch(int bn_tile, int kps, int cg, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                  const Params& p, cudaStream_t s, int mcast = 1) {
  if (mcast > 1) {  // A-multicast clusters (1-CTA MMAs, one reduce block per stage)
    if (cg == 1 && kps == 2 && bn_tile == 64) {
      if (mcast == 2) return launch_cfg<64, 4, 2, 0, 1, 2>(ma, mb, mc, p, s);
      if (mcast == 4) return launch_cfg<64, 4, 2, 0, 1, 4>(ma, mb, mc, p, s);
    }
    return fail(TPP_E_UNSUPPORTED, "no A-multicast kernel instantiation for this tile shape");
  }
  if (cg == 2) {
    if (kps == 1) {
      switch (bn_tile) {
        case 64: return launch_cfg<64, 8, 1, 0, 2>(ma, mb, mc, p, s);
        case 128: return launch_cfg<128, 8, 1, 0, 2>(ma, mb, mc, p, s);
        case 256: return launch_cfg<256, 6, 1, 0, 2>(ma, mb, mc, p, s);
      }
    } else if (kps == 2) {
      switch (bn_tile) {
        case 64: return launch_cfg<64, 4, 2, 0, 2>(ma, mb, mc, p, s);
        case 128: return launch_cfg<128, 4, 2, 0, 2>(ma, mb, mc, p, s);
        case 256: return launch_cfg<256, 3, 2, 0, 2>(ma, mb, mc, p, s);
      }
    } else if (kps == 4) {
      switch (bn_tile) {
        case 64: return launch_cfg<64, 2, 4, 0, 2>(ma, mb, mc, p, s);
      }
    }
    return fail(TPP_E_UNSUPPORTED, "no CTA-pair kernel instantiation for this tile width / stage depth");
  }
  if (kps == 1) {
    switch (bn_tile) {
      case 64: return launch_cfg<64, 8, 1>(ma, mb, mc, p, s);
      case 128: return launch_cfg<128, 6, 1>(ma, mb, mc, p, s);
      case 256: return launch_cfg<256, 4, 1>(ma, mb, mc, p, s);
    }
  } else if (kps == 2) {
    switch (bn_tile) {
      case 64: return launch_cfg<64, 4, 2>(ma, mb, mc, p, s);
      case 128: return launch_cfg<128, 3, 2>(ma, mb, mc, p, s);
      case 256: return launch_cfg<256, 2, 2>(ma, mb, mc, p, s);
    }
  } else if (kps == 4) {
    switch (bn_tile) {
      case 64: return launch_cfg<64, 2, 4>(ma, mb, mc, p, s);
    }
  } else if (kps == -1) {
    // B resident (conv weights), A-only stages, two producers
    switch (bn_tile) {
      case 64: return launch_cfg<64, 7, 1, 1>(ma, mb, mc, p, s);
    }
  } else if (kps == -2) {
    // B resident + one input halo per channel block (conv)
    switch (bn_tile) {
      case 64: return launch_cfg<64, 3, 1, 2>(ma, mb, mc, p, s);
    }
  } else if (kps == -3) {
    // as -2 with 4-row tiles (two accumulators per tile, 6-row halos)
    switch (bn_tile) {
      case 64: return launch_cfg<64, 2, 1, 3>(ma, mb, mc, p, s);
    }
  } else if (kps == -4) {
    // strips: 256 consecutive Wq-stride positions per tile, one halo box
    switch (bn_tile) {
      case 64: return launch_cfg<64, 2, 1, 4>(ma, mb, mc, p, s);
    }
  }
  return fail(TPP_E_UNSUPPORTED, "no kernel instantiation for this tile width / stage depth");
}

}  // namespace tc

int make_tma_map_5d(CUtensorMap* m, const void* base, const uint64_t dims[5], const uint64_t strides[4],
                    const uint32_t box[5], int swizzle_bytes) {
  const CUtensorMapSwizzle swz = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                 : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                       : CU_TENSOR_MAP_SWIZZLE_NONE;
  return tc::make_map_5d(m, base, dims, strides, box, swz);
}

int make_tma_map_5d_u8(CUtensorMap* m, const void* base, const uint64_t dims[5], const uint64_t strides[4],
                       const uint32_t box[5]) {
  return tc::make_map_5d(m, base, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_DATA_TYPE_UINT8);
}

// ---------------------------------------------------------------------------
// Blocked FC GEMMs on tensor cores.  Reference naming (kernels.py:287-297):
//   weights packed [m_b][k_b][bm][bk] (K-major), input [n_b][k_b][bn][bk],
//   output [n_b][m_b][bn][bm].
//   forward          out[t, f] = sum_c x[t, c]  W[f, c]      A K-major,  B K-major
//   backward-data    dx[t, c]  = sum_f dy[t, f] W[f, c]      A K-major,  B MN-major
//   backward-weights dW[f, c]  = sum_t dy[t, f] x[t, c]      A MN-major, B MN-major
// All three read the same blocked buffers in place — no transposes.  A
// pipeline stage carries KPS consecutive 64-wide reduce blocks in ONE TMA box
// per operand (the tensor-map dimension order puts the reduce-block index
// outermost in the box), so the single producer thread issues 2 TMA loads per
// KPS x 64 reduce elements.
// ---------------------------------------------------------------------------
namespace {

struct Operand {
  uint64_t dims[5];
  uint64_t strides[4];
  uint32_t box[5];
  tc::OpFeed feed;
};

// K-major operand: rows of a blocked [nblk][kblk][rows_b][k_in] tensor, tiles
// of `tile_rows` rows, `kps` reduce blocks per stage (kps > 1 needs k_in == 64).
Operand kmajor_operand(int nblk, int kblk, int rows_b, int k_in, int tile_rows, int kps) {
  Operand o{};
  const uint64_t kb = (uint64_t)k_in * 2;
  const bool split = rows_b >= tile_rows;
  const uint32_t box_rows = split ? tile_rows : rows_b, box_n = split ? 1 : tile_rows / rows_b;
  if (kps == 1) {
    o.dims[0] = 64; o.dims[1] = k_in / 64; o.dims[2] = rows_b; o.dims[3] = kblk; o.dims[4] = nblk;
    o.strides[0] = 128; o.strides[1] = kb; o.strides[2] = (uint64_t)rows_b * kb;
    o.strides[3] = (uint64_t)kblk * rows_b * kb;
    o.box[0] = 64; o.box[1] = 1; o.box[2] = box_rows; o.box[3] = 1; o.box[4] = box_n;
    o.feed = {2, 4, rows_b, tile_rows, 0, 1, k_in / 64, 0, 0};
  } else {
    // dims {c, 1, row, nblk, kblk}: the reduce block is the outermost box dim,
    // so one box = kps consecutive [tile_rows][64] K-major sub-tiles
    o.dims[0] = 64; o.dims[1] = 1; o.dims[2] = rows_b; o.dims[3] = nblk; o.dims[4] = kblk;
    o.strides[0] = 128; o.strides[1] = 128; o.strides[2] = (uint64_t)kblk * rows_b * 128;
    o.strides[3] = (uint64_t)rows_b * 128;
    o.box[0] = 64; o.box[1] = 1; o.box[2] = box_rows; o.box[3] = box_n; o.box[4] = kps;
    o.feed = {2, 3, rows_b, tile_rows, 1, kps, 0, tile_rows * 128, 0};
  }
  return o;
}

// MN-major operand over a blocked [red_blk][mn_blk][red_in][64] tensor (the
// MN block is exactly 64 wide = one 128B atom), tiles of `tile_mn` MN elements.
Operand mnmajor_operand(int red_blk, int mn_blk, int red_in, int tile_mn, int kps) {
  Operand o{};
  o.dims[0] = 64; o.dims[1] = red_in; o.dims[2] = mn_blk; o.dims[3] = red_blk; o.dims[4] = 1;
  o.strides[0] = 128; o.strides[1] = (uint64_t)red_in * 128; o.strides[2] = (uint64_t)mn_blk * red_in * 128;
  o.strides[3] = (uint64_t)red_blk * mn_blk * red_in * 128;
  o.box[0] = 64; o.box[2] = tile_mn / 64; o.box[4] = 1;
  if (red_in % (64 * kps) == 0) {
    // kps x 64 reduce rows inside one red block: smem [mn_local][64*kps][64]
    o.box[1] = 64 * kps; o.box[3] = 1;
    o.feed = {0, 2, 64, tile_mn, 0, 64 * kps, red_in, 64 * 128, 64 * kps * 128};
  } else {
    // red_in == 64: kps red blocks per box: smem [red_local][mn_local][64][64]
    o.box[1] = 64; o.box[3] = kps;
    o.feed = {0, 2, 64, tile_mn, kps == 1 ? 0 : 2, kps == 1 ? 64 : kps, red_in, (tile_mn / 64) * 64 * 128,
              64 * 128};
  }
  return o;
}

// experiment / diagnostic switches, read once per process
int env_dbg_mode() {
  static const int v = getenv("TPP_DBG_MODE") ? atoi(getenv("TPP_DBG_MODE")) : 0;
  return v;
}
int env_dbg_tile() {
  static const int v = getenv("TPP_DBG_TILE") ? atoi(getenv("TPP_DBG_TILE")) : 0;
  return v;
}
bool env_no_tma_store() {
  static const bool v = getenv("TPP_NO_TMA_STORE") != nullptr;
  return v;
}

int pick_bn(int feats, int tiles_m, int pref) {
  if (pref) return pref;
  static const int forced = [] {  // experiments: 64 / 128 / 256 only
    const int v = getenv("TPP_BN") ? atoi(getenv("TPP_BN")) : 0;
    return (v == 64 || v == 128 || v == 256) ? v : 0;
  }();
  if (forced && feats % forced == 0) return forced;
  int BN = 256;
  while (BN > 64 && (feats % BN != 0 || (int64_t)tiles_m * (feats / BN) < num_sms())) BN /= 2;
  return BN;
}

// reduce blocks per stage: as many as the smem budget of the tile allows
int pick_kps(int BN, int kblocks, bool kmajor_ok, int cg) {
  if (!kmajor_ok) return 1;
  static const int forced = [] {
    const char* e = getenv("TPP_KPS");  // tuning experiments only
    return e ? atoi(e) : 0;
  }();
  if (forced == 1 || forced == 2 || forced == 4) {
    if (kblocks % forced == 0 && !(forced == 4 && BN != 64)) return forced;
  }
  // 1-CTA wide tiles: keep the deeper pipeline (48 KB per block already);
  // pairs: 32 KB per block, two per TMA box halve the producer's issue count
  if (BN == 256) return (cg == 2 && kblocks % 2 == 0) ? 2 : 1;
  // BN = 64: two blocks per box (cfg 2: 6.25 us vs 6.7 us with four, 8.2 with one)
  if (kblocks % 2 == 0) return 2;
  return 1;
}

// CTAs per MMA: pairs (cta_group::2) when there are row tiles to pair up and
// each CTA's half of B is a whole swizzle atom for the operand's major-ness
int pick_cg(int BN, int tiles_m, int tiles_n, bool b_mn) {
  static const int forced = [] {
    const char* e = getenv("TPP_CG");  // tuning experiments only
    return e ? atoi(e) : 0;
  }();
  const bool ok = tiles_m >= 2 && (b_mn ? (BN / 2) % 64 == 0 : (BN / 2) % 32 == 0);
  if (forced == 1 || !ok) return 1;
  if (forced == 2) return 2;
  // wide tiles with at least a full wave of pairs: halve per-SM operand traffic
  return (BN == 256 && (int64_t)((tiles_m + 1) / 2) * tiles_n >= num_sms() / 2) ? 2 : 1;
}

// Long GEMMs with less than a wave of pair tiles: one wave of 256-wide pair
// tiles (the tensor pipe at its floor) can beat ~2 waves of 1-CTA tiles that
// are shared-memory bound (128 x 128: both 4 KB operands per 64-cycle MMA; 128
// x 256: 188 B/cycle; 128 x 64: 48-cycle MMAs).  Cost per SM ~ waves x the
// SM's share of a tile / MMA efficiency; measured on the cfg-5 dW of the
// 1024-wide layers (1024 x 4096 over 8192 tokens): 79 us as 64 pair tiles in
// one wave vs 102 us as 256 1-CTA 128 x 128 tiles in 1.73 waves.
void prefer_pairs(int feats, int tiles_m, int pref, int& BN, int& cg, int blk = 64) {
  static const bool forced = getenv("TPP_BN") != nullptr || getenv("TPP_CG") != nullptr;
  if (cg == 2 || pref || forced || feats % 256 != 0 || tiles_m < 2) return;
  if (blk >= 256 ? blk % 256 != 0 : 256 % blk != 0) return;  // output blocks must tile the 256-wide tile
  auto eff = [](int bn) { return bn == 256 ? 0.68 : bn == 128 ? 0.77 : 0.67; };
  const int64_t sms = num_sms(), pairs = sms / 2;
  const int64_t u1 = (int64_t)tiles_m * (feats / BN), w1 = (u1 + sms - 1) / sms;
  const int64_t u2 = (int64_t)((tiles_m + 1) / 2) * (feats / 256), w2 = (u2 + pairs - 1) / pairs;
  const double c1 = (double)w1 * 128.0 * BN / eff(BN), c2 = (double)w2 * 128.0 * 256.0;
  if (c2 < c1) {
    BN = 256;
    cg = 2;
  }
}

// A-multicast cluster size for forward FC (experiments: TPP_MC=2|4).  Off by
// default: on cfg 2 (one 128x64 tile per CTA) clusters of 2 / 4 sharing the
// activation boxes measured 6.96 / 7.12 us against 6.25 us without -- halving
// the per-SM A bytes does not pay for coupling every stage to the slowest CTA.
int pick_mc(int BN, int cg, int kps, int tiles_m, int tiles_n) {
  static const int forced = [] {
    const char* e = getenv("TPP_MC");
    return e ? atoi(e) : 0;
  }();
  if (BN != 64 || cg != 1 || kps != 2 || (forced != 2 && forced != 4)) return 1;
  (void)tiles_m;
  return tiles_n % forced == 0 ? forced : 1;
}

int run_gemm(const Operand& A, const Operand& B, const void* a_ptr, const void* b_ptr, tc::Params p,
             int BN, int kps, int cg, cudaStream_t stream, int mcast = 1) {
  CUtensorMap ma, mb, mc;
  int rc = tc::make_map_5d(&ma, a_ptr, A.dims, A.strides, A.box);
  if (rc) return rc;
  rc = tc::make_map_5d(&mb, b_ptr, B.dims, B.strides, B.box);
  if (rc) return rc;
  // BF16 outputs leave through smem staging + TMA stores: output tensor
  // [ntb][o_mb][o_bn][o_bm], box = 32 tokens x 32 features, 64B swizzle
  p.tma_store = !env_no_tma_store() && !(p.flags & (TPP_FC_OUT_FP32 | TPP_FC_SGD)) && p.o_bn % 32 == 0 && p.o_bm % 32 == 0 &&
                reinterpret_cast<uintptr_t>(p.out) % 16 == 0;
  mc = ma;
  if (p.tma_store) {
    const uint64_t rowb = (uint64_t)p.o_bm * 2;
    const uint64_t dims[5] = {(uint64_t)p.o_bm, 1, (uint64_t)p.o_bn, (uint64_t)p.o_mb,
                              (uint64_t)((p.tokens + p.o_bn - 1) / p.o_bn)};
    const uint64_t str[4] = {rowb, rowb, (uint64_t)p.o_bn * rowb, (uint64_t)p.o_mb * p.o_bn * rowb};
    const uint32_t box[5] = {32, 1, 32, 1, 1};
    rc = tc::make_map_5d(&mc, p.out, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
  p.fa = A.feed;
  p.fb = B.feed;
  return tc::launch(BN, kps, cg, ma, mb, mc, p, stream, mcast);
}

}  // namespace

// flavor: 0 forward, 1 backward-data, 2 backward-weights
static unsigned long long* g_dbg_ts = nullptr;
void set_debug_timestamps(unsigned long long* p) { g_dbg_ts = p; }
unsigned long long* debug_timestamps() { return g_dbg_ts; }

int fc_gemm_tc(int flavor, const tpp_fc_desc* d, const void* w_packed, const void* x_or_dy,
               const void* x_for_dw, const void* bias, const void* residual, void* out,
               void* mask_out, const void* mask_in, cudaStream_t stream, uint16_t* sgd_lo, float sgd_lr) {
  using namespace tc;
  const int m_b = d->m_b, n_b = d->n_b, k_b = d->k_b, bm = d->bm, bn = d->bn, bk = d->bk;
  Params p{};
  p.sgd_lo = sgd_lo;
  p.sgd_lr = sgd_lr;
  p.mode = FEED_FC;
  p.act = d->activation;
  p.flags = d->flags;
  p.bias = bias;
  p.residual = reinterpret_cast<const uint16_t*>(residual);
  p.out = out;
  p.mask = reinterpret_cast<uint8_t*>(mask_out);
  p.mask_in = reinterpret_cast<const uint8_t*>(mask_in);
  p.dbg = g_dbg_ts;
  p.dbg_tile = g_dbg_ts ? env_dbg_tile() : 0;
  p.dbg_mode = env_dbg_mode();
  TPP_REQUIRE((bn < BM && BM % bn == 0) || (bn >= BM && bn % BM == 0), TPP_E_UNSUPPORTED,
              "tensor-core FC needs bn | 128 or 128 | bn");
  if (flavor == 0) {
    TPP_REQUIRE(bk % 64 == 0 && bm % 32 == 0, TPP_E_UNSUPPORTED, "tensor-core FC needs bk % 64 == 0, bm % 32 == 0");
    const int feats = m_b * bm, tokens = n_b * bn;
    const int tiles_m = (tokens + BM - 1) / BM;
    int BN = pick_bn(feats, tiles_m, d->block_n);
    TPP_REQUIRE(feats % BN == 0 && ((bm >= BN && bm % BN == 0) || (bm < BN && BN % bm == 0)),
                TPP_E_UNSUPPORTED, "features must tile by the tile width");
    const int kblocks = k_b * (bk / 64);
    int cg = pick_cg(BN, tiles_m, feats / BN, false);
    prefer_pairs(feats, tiles_m, d->block_n, BN, cg, bm);
    const int kps = pick_kps(BN, kblocks, bk == 64, cg);
    const int mc = pick_mc(BN, cg, kps, tiles_m, feats / BN);
    p.tokens = tokens; p.kblocks = kblocks;
    p.tiles_m = tiles_m; p.tiles_n = feats / BN; p.feats = feats; p.bn_tile = BN;
    p.o_bn = bn; p.o_bm = bm; p.o_mb = m_b;
    return run_gemm(kmajor_operand(n_b, k_b, bn, bk, BM, kps), kmajor_operand(m_b, k_b, bm, bk, BN / cg, kps),
                    x_or_dy, w_packed, p, BN, kps, cg, stream, mc);
  }
  if (flavor == 1) {
    // dx[n_b][k_b][bn][bk] = dy[n_b][m_b][bn][bm] . W ; B = W as MN-major over its bk
    TPP_REQUIRE(bk == 64 && bm % 64 == 0, TPP_E_UNSUPPORTED, "backward-data needs bk == 64, bm % 64 == 0");
    const int feats = k_b * bk, tokens = n_b * bn;
    const int tiles_m = (tokens + BM - 1) / BM;
    int BN = pick_bn(feats, tiles_m, d->block_n);
    TPP_REQUIRE(feats % BN == 0, TPP_E_UNSUPPORTED, "input features must tile by the tile width");
    const int kblocks = m_b * (bm / 64);
    int cg = pick_cg(BN, tiles_m, feats / BN, true);
    prefer_pairs(feats, tiles_m, d->block_n, BN, cg);
    const int kps = pick_kps(BN, kblocks, bm == 64, cg);
    p.tokens = tokens; p.kblocks = kblocks;
    p.tiles_m = tiles_m; p.tiles_n = feats / BN; p.feats = feats; p.bn_tile = BN;
    p.o_bn = bn; p.o_bm = bk; p.o_mb = k_b;
    p.b_mn = 1;
    return run_gemm(kmajor_operand(n_b, m_b, bn, bm, BM, kps), mnmajor_operand(m_b, k_b, bm, BN / cg, kps), x_or_dy,
                    w_packed, p, BN, kps, cg, stream);
  }
  // flavor 2: dW[m_b][k_b][bm][bk] = sum_t dy[t][f] x[t][c]
  TPP_REQUIRE(bm == 64 && bk == 64 && bn % 64 == 0, TPP_E_UNSUPPORTED,
              "backward-weights needs bm == bk == 64 and bn % 64 == 0");
  const int rows = m_b * bm, feats = k_b * bk;
  const int tiles_m = (rows + BM - 1) / BM;
  int BN = pick_bn(feats, tiles_m, d->block_n);
  TPP_REQUIRE(feats % BN == 0, TPP_E_UNSUPPORTED, "input features must tile by the tile width");
  const int kblocks = n_b * (bn / 64);
  int cg = pick_cg(BN, tiles_m, feats / BN, true);
  prefer_pairs(feats, tiles_m, d->block_n, BN, cg);
  int kps = pick_kps(BN, kblocks, true, cg);
  while (kps > 1 && bn != 64 && bn % (64 * kps) != 0) kps /= 2;  // a box must not skip token rows
  p.tokens = rows; p.kblocks = kblocks;
  p.tiles_m = tiles_m; p.tiles_n = feats / BN; p.feats = feats; p.bn_tile = BN;
  p.o_bn = bm; p.o_bm = bk; p.o_mb = k_b;
  p.a_mn = 1; p.b_mn = 1;
  return run_gemm(mnmajor_operand(n_b, m_b, bn, BM, kps), mnmajor_operand(n_b, k_b, bn, BN / cg, kps), x_or_dy,
                  x_for_dw, p, BN, kps, cg, stream);
}

int fc_forward_tc(const tpp_fc_desc* d, const void* w_packed, const void* x, const void* bias,
                  const void* residual, void* out, void* mask, cudaStream_t stream) {
  return fc_gemm_tc(0, d, w_packed, x, nullptr, bias, residual, out, mask, nullptr, stream);
}

// ---------------------------------------------------------------------------
// 3x3 (R x S) stride-1 'same' convolution, bc = bk = 64 per block.
//   input [N][C_b][H][W][64], weights packed [K_b][R][S][C_b][64 out][64 in],
//   output [N][K_b][H][W][64].  Tiles: 2 output rows x 64 columns (W <= 64).
// ---------------------------------------------------------------------------
int conv_forward_tc(int N, int Cb, int Kb, int H, int W, int R, int S, int pad,
                    const void* w_packed, const void* x, void* out, cudaStream_t stream) {
  using namespace tc;
  TPP_REQUIRE(W <= 64, TPP_E_UNSUPPORTED, "tensor-core conv tiles need W <= 64");
  TPP_REQUIRE(2 * pad == R - 1 && 2 * pad == S - 1, TPP_E_UNSUPPORTED,
              "tensor-core conv implements 'same' padding");
  const int P = H, Q = W;
  const int feats = Kb * 64;
  const int BN = feats >= 256 && feats % 256 == 0 ? 256 : (feats % 128 == 0 ? 128 : 64);
  Params p{};
  p.mode = FEED_CONV;
  p.dbg = g_dbg_ts;
  p.dbg_mode = env_dbg_mode();
  p.kblocks = R * S * Cb;
  p.cv_P = P;
  p.cv_Q = Q;
  p.cv_R = R;
  p.cv_S = S;
  p.cv_pad = pad;
  p.cv_Cb = Cb;
  // output rows per tile: 4 (RES 3) when the halo path and TMA stores apply
  static const bool two_row = getenv("TPP_CONV_2ROW") != nullptr;  // experiments
  const bool res_ok = BN == 64 && feats / BN == 1 && (int64_t)p.kblocks * BN * 128 <= tc::kResMaxBytes;
  const bool halo_ok = res_ok && 2 + R - 1 <= tc::kHaloRows && W + S - 1 <= 64;
  const bool rows4 = halo_ok && !two_row && reinterpret_cast<uintptr_t>(out) % 16 == 0 && !env_no_tma_store();
  // strips (RES 4): 3x3, pad 1, Wq = W + 1 <= 64, 16-byte aligned output
  static const bool no_strip = getenv("TPP_CONV_ROWS") != nullptr;  // experiments: the row tiles
  const int wq = W + pad;
  const int strip_hr = (wq - 1 + 2 * BM + (R - 1) * wq + (S - 1) + wq - 1) / wq;
  const bool strip = res_ok && !no_strip && R == 3 && S == 3 && pad == 1 && wq <= 64 &&
                     strip_hr * wq * 128 <= tc::kStripHaloBytes && reinterpret_cast<uintptr_t>(out) % 32 == 0;
  p.cv_rows = rows4 ? 4 : 2;
  p.cv_tiles_per_img = (P + p.cv_rows - 1) / p.cv_rows;
  if (strip) {
    p.cv_wq = wq;
    p.cv_tiles_per_img = (P * wq + 2 * BM - 1) / (2 * BM);
    p.stage_tx = strip_hr * wq * 128;
  }
  p.tiles_m = N * p.cv_tiles_per_img;
  p.tiles_n = feats / BN;
  p.feats = feats;
  p.bn_tile = BN;
  p.o_bn = P * Q;
  p.o_bm = 64;
  p.o_mb = Kb;
  p.act = TPP_ACT_NONE;
  p.flags = 0;
  p.out = out;

  const bool res = BN == 64 && p.tiles_n == 1 && (int64_t)p.kblocks * BN * 128 <= tc::kResMaxBytes;
  // halo: one box of (2 + R - 1) input rows x 64 pixels per channel block
  const bool halo = res && 2 + R - 1 <= tc::kHaloRows && W + S - 1 <= 64;
  CUtensorMap ma, mb, mc;
  {
    const uint64_t dims[5] = {64, (uint64_t)W, (uint64_t)H, (uint64_t)Cb, (uint64_t)N};
    const uint64_t str[4] = {128, (uint64_t)W * 128, (uint64_t)H * W * 128, (uint64_t)Cb * H * W * 128};
    uint32_t box[5] = {64, 64, halo ? (uint32_t)(p.cv_rows + 2) : 2u, 1, 1};
    if (strip) {  // rows of Wq pixels from x = -pad: adjacent rows share the pad column
      box[1] = (uint32_t)wq;
      box[2] = (uint32_t)strip_hr;
    }
    int rc = make_map_5d(&ma, x, dims, str, box);
    if (rc) return rc;
  }
  // output [N][K_b][H][W][64] through TMA stores: box 32 channels x 32 pixels
  // (strips store from registers)
  p.tma_store = !strip && reinterpret_cast<uintptr_t>(out) % 16 == 0 && !env_no_tma_store();
  mc = ma;
  if (p.tma_store) {
    const uint64_t dims[5] = {64, (uint64_t)W, (uint64_t)H, (uint64_t)Kb, (uint64_t)N};
    const uint64_t str[4] = {128, (uint64_t)W * 128, (uint64_t)H * W * 128, (uint64_t)Kb * H * W * 128};
    const uint32_t box[5] = {32, 32, 1, 1, 1};
    int rc = make_map_5d(&mc, out, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
  // weights: K-major rows [K_b][J = R*S*C_b][64 out][64 in]
  const Operand wb = kmajor_operand(Kb, R * S * Cb, 64, 64, BN, 1);
  p.fb = wb.feed;
  {
    int rc = make_map_5d(&mb, w_packed, wb.dims, wb.strides, wb.box);
    if (rc) return rc;
  }
  return launch(BN, strip ? -4 : halo ? (rows4 ? -3 : -2) : (res ? -1 : 1), 1, ma, mb, mc, p, stream);
}

}  // namespace tpp

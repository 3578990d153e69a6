// EXPERIMENT (not built; kept for the record, see DESIGN.md §4 "conv tap stacking").
// Measured on B200 (cfg 4 forward, 256 x 56 x 56, C = K = 64): N = 192 tap
// stacking -- MMA pipeline alone 43 us (82 % of burst), but the epilogue's
// lane shifts (two shuffles per output, a cross-quarter exchange) and the
// scattered output stores on the shared L1/smem port made the whole kernel
// 87-89 us; N = 128 (taps 0, 1) + N = 64 (tap 2): MMA alone 52.7 us, whole
// 72.5 us -- vs 70-72 us for the halo kernel in brgemm_tc.cu, so the halo
// kernel stays.  To build it, add it to _build.SOURCES and route
// conv_forward_tc through conv3x3_tap_tc.
// K2n: 3x3 'same' convolution (stride 1, C = K = 64 channels per image) with
// the filter taps of one kernel row stacked along the MMA N dimension.
//
// The halo kernel in brgemm_tc.cu issues one M=128 x N=64 MMA per (tap, 16
// channels): 6 KB of shared-memory operand reads per 131k MACs, 48 cycles each
// (the shared-memory port is the bound, tensor pipe ~50 % active).  Here the
// B operand of one MMA is the three taps (r, 0), (r, 1), (r, 2) of a kernel
// row stacked along N (192 rows of the resident K-major weights, which the
// packed layout [R][S][64 out][64 in] already holds contiguously), and A is
// the input halo viewed from the row of tap (r, 0): M=128 x N=192 x K=16,
// 10 KB per 393k MACs at the tensor pipe's N=192 rate (96 cycles) -- 2.2x
// fewer operand bytes per MAC.  Column block s of the accumulator row for
// position p then holds tap (r, s)'s contribution to output position p - s,
// so the epilogue adds
//     out[p] = (D[p][0:64] + D[p+1][64:128]) + D[p+2][128:192]
// with two warp shuffles per value (the two positions past each 32-lane
// quarter come from the next quarter through shared memory).  A tile is 128
// consecutive positions of the W+1-stride position space (the right pad
// column of input row y is the left pad of row y + 1; one TMA box of 6 input
// rows x (W + 1) pixels, OOB zero fill = padding) and produces 126 outputs.
//
// Roles (one persistent CTA per SM): warp 0 TMA producer, warp 1 MMA issuer,
// warp 2 TMEM allocator, warps 4-11 epilogue (quarter q = TMEM lanes 32q..,
// half hh = output channels 32hh..).  TMEM: two 192-column accumulators.

#include <cstdlib>
#include <cuda.h>

#include "common.cuh"
#include "sm100.cuh"

namespace tpp {

using namespace sm100;

namespace ctap {

constexpr int kEpiWarp0 = 4;
constexpr int kEpiWarps = 16;         // 4 per TMEM lane quarter, 16 output channels each
constexpr int kCh = 64 / (kEpiWarps / 4);
constexpr int kThreads = 32 * (kEpiWarp0 + kEpiWarps);
constexpr int kPos = 128;             // MMA M: positions per tile
constexpr int kOut = kPos - 1;        // outputs per tile (the last one needs the next tile's row)
constexpr int kStages = 3;
constexpr int kWBytes = 3 * 192 * 128;  // resident weights: 3 kernel rows x 192 rows x 64 bf16
constexpr int kNBuf = 4;
constexpr int kAccCols = 128;
constexpr int kXchFloats = kCh;       // per warp: lane 0's tap-(r, 1) block, kCh channels

struct Params {
  int N, P, Q, wq;        // images, output rows / cols, position-row stride Q + 1
  int tiles_per_img, tiles;
  int stage_bytes, halo_tx, halo_rows;
  void* out;              // [N][1][P][Q][64] bf16
  int dbg;                // experiments (TPP_CONV_DBG): bit 0 no epilogue math / stores, bit 1 no MMAs,
                          // bit 2 no stores, bit 3 no exchange barrier
};

__host__ __device__ constexpr int stage_alloc(int halo_bytes) { return (halo_bytes + 1023) & ~1023; }

__global__ void __launch_bounds__(kThreads, 1)
conv3x3_tap_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                   const Params p) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* wres = smem;                                   // kWBytes, 1024-aligned
  uint8_t* halo = smem + kWBytes;                         // kStages x stage_bytes
  // the epilogue's exchange slots [2][8 warps][96] (static: the compiler then
  // knows they are shared memory -- generic loads / stores otherwise)
  __shared__ __align__(16) float xch[2 * kEpiWarps * kXchFloats];
  uint64_t* bars = reinterpret_cast<uint64_t*>(halo + kStages * p.stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + kNBuf;
  uint64_t* bres = tempty + kNBuf;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres + 1);

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&map_x);
    prefetch_tmap(&map_w);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < kNBuf; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    mbar_init(bres, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      mbar_arrive_expect_tx(bres, kWBytes);
      for (int r = 0; r < 3; ++r) tma_load_5d(wres + r * 192 * 128, &map_w, bres, 0, 0, r, 0, 0);
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        const int img = tile / p.tiles_per_img;
        const int p0 = (tile - img * p.tiles_per_img) * kOut;
        const int y0 = p0 / p.wq;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], (uint32_t)p.halo_tx);
        // input rows y0 - 1 .., pixels -1 .. Q - 1 (OOB zero fill = padding)
        tma_load_5d(halo + s * p.stage_bytes, &map_x, &full[s], 0, -1, y0 - 1, 0, img);
        if (++s == kStages) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (warp-collective, one elected lane) =====================
    const uint32_t idesc2 = idesc_bf16_f32(kPos, 128), idesc1 = idesc_bf16_f32(kPos, 64);
    const uint64_t wdesc0 = sw128_kmajor_desc(smem_u32(wres));
    const uint64_t hdesc0 = sw128_kmajor_desc(smem_u32(halo));
    mbar_wait(bres, 0);
    int s = 0;
    uint32_t ph = 0, tcount = 0;
    for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x, ++tcount) {
      const int img = tile / p.tiles_per_img;
      const int p0 = (tile - img * p.tiles_per_img) * kOut;
      const uint32_t off = (uint32_t)(p0 - (p0 / p.wq) * p.wq);   // halo row of the tile's first position
      const uint32_t b = tcount % kNBuf, bph = (tcount / kNBuf) & 1;
      mbar_wait(&tempty[b], bph ^ 1);
      tc_fence_after();
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + b * kAccCols;
      // descriptor start addresses are in 16-byte units: a 128-byte halo row is 8
      const uint64_t a0 = hdesc0 + (uint64_t)((s * p.stage_bytes) >> 4) + (uint64_t)off * 8;
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const uint64_t ar = a0 + (uint64_t)(r * p.wq) * 8;
        const uint64_t br = wdesc0 + (uint64_t)((r * 192 * 128) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (p.dbg & 2) continue;
          // taps (r, 0), (r, 1) stacked along N from the row of tap (r, 0) ...
          umma_f16_warp(tmem_d, ar + 2 * kk, br + 2 * kk, idesc2, (r > 0 || kk > 0) ? 1u : 0u);
          // ... and tap (r, 2) from its own row, straight into block 0
          umma_f16_warp(tmem_d, ar + 16 + 2 * kk, br + (128 * 128 >> 4) + 2 * kk, idesc1, 1u);
        }
      }
      umma_commit_warp(&empty[s]);
      umma_commit_warp(&tfull[b]);
      if (++s == kStages) { s = 0; ph ^= 1; }
    }
  } else if (warp >= kEpiWarp0) {
    // ===================== epilogue =====================
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int ew = warp - kEpiWarp0;
    const int q = warp & 3;       // TMEM lane quarter of this warp
    const int hh = ew >> 2;       // output channels kCh hh .. kCh hh + kCh - 1
    uint32_t tcount = 0;
    for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x, ++tcount) {
      const int img = tile / p.tiles_per_img;
      const int p0 = (tile - img * p.tiles_per_img) * kOut;
      const int pl = q * 32 + lane;          // position within the tile
      const int pos = p0 + pl;
      const int oy = pos / p.wq, ox = pos - oy * p.wq;
      const uint32_t b = tcount % kNBuf, bph = (tcount / kNBuf) & 1;
      mbar_wait(&tfull[b], bph);
      tc_fence_after();
      const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + b * kAccCols + hh * kCh;
      uint32_t v0[kCh], v1[kCh];
      tmem_ld16(ta, v0);
      tmem_ld16(ta + 64, v1);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
      if (p.dbg & 1) continue;
      // the next quarter's first lanes, for this quarter's last two positions
      float* xw = xch + ((tcount & 1) * kEpiWarps + ew) * kXchFloats;
      if (lane == 0) {
#pragma unroll
        for (int c = 0; c < kCh; ++c) xw[c] = __uint_as_float(v1[c]);
      }
      if (!(p.dbg & 8)) named_bar_sync(1, kEpiWarps * 32);
      const float* xn = xch + ((tcount & 1) * kEpiWarps + (hh * 4 + ((q + 1) & 3))) * kXchFloats;
      float o[kCh];
      {
        // lane 31: the next quarter's lane 0 (broadcast loads, no divergence)
        float e1[kCh];
#pragma unroll
        for (int c = 0; c < kCh; c += 4) {
          const float4 t4 = *reinterpret_cast<const float4*>(xn + c);
          e1[c] = t4.x; e1[c + 1] = t4.y; e1[c + 2] = t4.z; e1[c + 3] = t4.w;
        }
#pragma unroll
        for (int c = 0; c < kCh; ++c) {
          float s1 = __uint_as_float(v1[c]);
          if (!(p.dbg & 16)) s1 = __shfl_down_sync(0xffffffffu, s1, 1);
          s1 = lane == 31 ? e1[c] : s1;
          o[c] = __fadd_rn(__uint_as_float(v0[c]), s1);
        }
      }
      if (pl < kOut && ox < p.Q && oy < p.P && !(p.dbg & 4)) {
        uint32_t w[kCh / 2];
        pack_bf16_ref_n<kCh / 2>(o, w);
        // two 256-bit stores (full 32-byte sectors): the epilogue's global
        // stores are otherwise the kernel's bottleneck (16-byte pieces of 32
        // different lines per warp instruction)
        uint16_t* op = reinterpret_cast<uint16_t*>(p.out) + (((int64_t)img * p.P + oy) * p.Q + ox) * 64 + hh * kCh;
#pragma unroll
        for (int i = 0; i < kCh / 16; ++i)
          asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(op + 16 * i), "r"(w[8 * i]),
                       "r"(w[8 * i + 1]), "r"(w[8 * i + 2]), "r"(w[8 * i + 3]), "r"(w[8 * i + 4]), "r"(w[8 * i + 5]),
                       "r"(w[8 * i + 6]), "r"(w[8 * i + 7])
                       : "memory");
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace ctap

// 1 = not applicable (the caller runs the halo kernel)
int conv3x3_tap_tc(int N, int Cb, int Kb, int H, int W, int R, int S, int pad, const void* w_packed,
                   const void* x, void* out, cudaStream_t stream) {
  using namespace ctap;
  static const bool off = getenv("TPP_CONV_HALO") != nullptr;  // A/B: the halo kernel
  if (off || Cb != 1 || Kb != 1 || R != 3 || S != 3 || pad != 1 || W + 1 > 256 || H < 1 || N < 1 ||
      reinterpret_cast<uintptr_t>(out) % 32 != 0)
    return 1;
  Params p{};
  p.N = N; p.P = H; p.Q = W; p.wq = W + 1;
  p.tiles_per_img = (H * p.wq + kOut - 1) / kOut;
  p.tiles = N * p.tiles_per_img;
  // rows a tile can touch: positions off .. off + 127 (off < wq) plus the taps' 2 wq
  p.halo_rows = (p.wq - 1 + kPos - 1 + 2 * p.wq) / p.wq + 1;
  p.halo_tx = p.halo_rows * p.wq * 128;
  p.stage_bytes = stage_alloc(p.halo_tx);
  p.out = out;
  static const int dbg = getenv("TPP_CONV_DBG") ? atoi(getenv("TPP_CONV_DBG")) : 0;
  p.dbg = dbg;
  CUtensorMap mx, mw;
  {
    const uint64_t dims[5] = {64, (uint64_t)W, (uint64_t)H, 1, (uint64_t)N};
    const uint64_t str[4] = {128, (uint64_t)W * 128, (uint64_t)H * W * 128, (uint64_t)H * W * 128};
    const uint32_t box[5] = {64, (uint32_t)p.wq, (uint32_t)p.halo_rows, 1, 1};
    int rc = make_tma_map_5d(&mx, x, dims, str, box, 128);
    if (rc) return rc;
  }
  {
    // packed weights [R=3][S=3][64 out][64 in]: kernel row r = 192 consecutive K-major rows
    const uint64_t dims[5] = {64, 192, 3, 1, 1};
    const uint64_t str[4] = {128, 192 * 128, 3 * 192 * 128, 3 * 192 * 128};
    const uint32_t box[5] = {64, 192, 1, 1, 1};
    int rc = make_tma_map_5d(&mw, w_packed, dims, str, box, 128);
    if (rc) return rc;
  }
  const size_t smem = 1024 + kWBytes + (size_t)kStages * p.stage_bytes + (2 * kStages + 2 * kNBuf + 1) * 8 + 16;
  if (smem + 2 * kEpiWarps * kXchFloats * sizeof(float) > 227 * 1024 || p.halo_rows > 256) return 1;
  cudaError_t e = ensure_smem_attr((const void*)conv3x3_tap_kernel, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(conv3x3_tap_kernel)");
  const int grid = p.tiles < num_sms() ? p.tiles : num_sms();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, conv3x3_tap_kernel, mx, mw, p);
  if (e != cudaSuccess) return cuda_status(e, "cudaLaunchKernelEx(conv3x3_tap_kernel)");
  TPP_CUDA_LAUNCH_CHECK("conv3x3_tap_kernel");
  set_last_config("conv3x3_tap_kernel grid=" + std::to_string(grid) + " tiles=" + std::to_string(p.tiles));
  return TPP_OK;
}

}  // namespace tpp

// Convolution backward-weights on tcgen05 (the training-side
// neighbour of the offset-BRGEMM forward).
//
//   dW[kb][cb][r][s][c][k] = sum_{n,p,q} X[n][cb][p+r-pad][q+s-pad][c] * dO[n][kb][p][q][k]
//
// a batch-reduce over pixels for every tap.  One CTA per SM owns a range of
// output rows (n, p) of one (kb, cb) block pair and keeps ALL taps'
// accumulators in TMEM for its whole range:
//
//   * per output row ONE TMA box of the input halo (R rows x 64 pixels x 64
//     channels, OOB zero fill = padding) and ONE box of dO (64 pixels x 64 k);
//   * the reduction dimension (pixels) is the MMA K; both operands are
//     MN-major (channels contiguous in 128-byte rows), so a tap's operand is
//     the halo viewed from row r*64 + s — a row-shifted SW128 descriptor;
//   * M = 128 covers TWO taps: the descriptor's second 64-wide M atom starts
//     LBO = (shift(t1) - shift(t0)) * 128 bytes after the first (the two views
//     overlap in shared memory, which the MMA only reads), N = 64 = dO's k.
//     9 taps -> 5 tap pairs (the last one repeats tap 7), 5 x 64 TMEM columns.
//
// Partials of the CTAs that split one (kb, cb) are summed by a second kernel in
// a fixed order (deterministic).

#include <cstdlib>
#include <cuda.h>

#include "common.cuh"
#include "sm100.cuh"

namespace tpp {

using namespace sm100;

namespace cdw {

constexpr int kThreads = 256;  // w0 producer, w1 MMA, w2 TMEM alloc, w4-7 epilogue
constexpr int kMaxR = 3;
constexpr int kHaloBytes = kMaxR * 64 * 128;  // 24 KB
constexpr int kDoBytes = 64 * 128;            // 8 KB
constexpr int kStageBytes = kHaloBytes + kDoBytes;
constexpr int kStages = 5;
constexpr int kMaxPairs = 8;

struct Params {
  int N, H, W, R, S, pad, Cb, Kb;
  int Z;          // CTAs per (kb, cb)
  int taps, pairs;
  float* partial; // [Kb*Cb*Z][taps][64 c][64 k]
};

// RS3 = 1: a 3x3 filter, every tap-pair descriptor offset an immediate (the
// single issuing warp must keep pace with 48-cycle N=64 MMAs)
template <int RS3>
__global__ void __launch_bounds__(kThreads, 1)
conv_dw_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_do, const Params p) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* done = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;  // warp-uniform (uniform-datapath MMA issue)

  const int item = blockIdx.x;
  const int kbcb = item / p.Z, z = item % p.Z;
  const int kb = kbcb / p.Cb, cb = kbcb % p.Cb;
  const int rows = p.N * p.H;
  const int r0 = (int)((int64_t)rows * z / p.Z), r1 = (int)((int64_t)rows * (z + 1) / p.Z);

  if (threadIdx.x == 0) {
    prefetch_tmap(&map_x);
    prefetch_tmap(&map_do);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // uniform (MMA operand)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int n = r0 / p.H, pr = r0 % p.H;
      for (int row = r0; row < r1; ++row) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * kStageBytes;
        mbar_arrive_expect_tx(&full[s], p.R * 64 * 128 + kDoBytes);
        // halo: input rows pr - pad .. pr - pad + R - 1, pixels -pad .. 63 - pad
        tma_load_5d(st, &map_x, &full[s], 0, -p.pad, pr - p.pad, cb, n);
        tma_load_5d(st + kHaloBytes, &map_do, &full[s], 0, 0, pr, kb, n);
        if (++pr == p.H) { pr = 0; ++n; }
        if (++s == kStages) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // the whole warp runs the issue loop; one elected lane issues
    const uint32_t idesc = idesc_bf16_f32(128, 64, 1, 1);
    int s = 0;
    uint32_t ph = 0;
    for (int row = r0; row < r1; ++row) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint32_t st = smem_u32(smem + s * kStageBytes);
      const uint64_t bdesc = sw128_mnmajor_desc(st + kHaloBytes, 8192);
      if (RS3) {
        const uint64_t a0 = sw128_mnmajor_desc(st, 0);
#pragma unroll
        for (int pp = 0; pp < 5; ++pp) {
          const int t0 = pp < 4 ? 2 * pp : 7, t1 = t0 + 1;
          const int sh0 = (t0 / 3) * 64 + t0 % 3, sh1 = (t1 / 3) * 64 + t1 % 3;
          // start address (16-byte units) and LBO field (bits 16..29) as immediates
          const uint64_t adesc = a0 + (uint64_t)((sh0 * 128) >> 4) + ((uint64_t)(((sh1 - sh0) * 128) >> 4) << 16);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_f16_warp(tmem_base + pp * 64, adesc + (uint64_t)(kk * (2048 >> 4)),
                          bdesc + (uint64_t)(kk * (2048 >> 4)), idesc, (row > r0 || kk > 0) ? 1u : 0u);
        }
      } else {
        for (int pp = 0; pp < p.pairs; ++pp) {
          const int t0 = pp * 2 < p.taps - 1 ? pp * 2 : p.taps - 2, t1 = t0 + 1;
          const int sh0 = (t0 / p.S) * 64 + t0 % p.S, sh1 = (t1 / p.S) * 64 + t1 % p.S;
          const uint64_t adesc = sw128_mnmajor_desc(st + sh0 * 128, (uint32_t)(sh1 - sh0) * 128);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_f16_warp(tmem_base + pp * 64, adesc + (uint64_t)(kk * (2048 >> 4)),
                          bdesc + (uint64_t)(kk * (2048 >> 4)), idesc, (row > r0 || kk > 0) ? 1u : 0u);
        }
      }
      umma_commit_warp(&empty[s]);
      if (++s == kStages) { s = 0; ph ^= 1; }
    }
    umma_commit_warp(done);
  } else if (warp >= 4) {
    // epilogue: TMEM lanes q*32.. = channels (q&1)*32.. of tap t0 (q < 2) or t1
    const int q = warp & 3;
    mbar_wait(done, 0);
    tc_fence_after();
    if (r1 > r0) {
      for (int pp = 0; pp < p.pairs; ++pp) {
        const int t0 = pp * 2 < p.taps - 1 ? pp * 2 : p.taps - 2;
        const bool dup = pp * 2 >= p.taps - 1 && (p.taps & 1);  // last pair of an odd tap count repeats t0
        const int tap = q < 2 ? t0 : t0 + 1;
        const int c = (q & 1) * 32 + lane;
        float* dst = p.partial + (((int64_t)item * p.taps + tap) * 64 + c) * 64;
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          uint32_t v[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + pp * 64 + half * 32, v);
          tmem_ld_wait();
          if (q < 2 && dup) continue;
          float4* o = reinterpret_cast<float4*>(dst + half * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            o[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]), __uint_as_float(v[4 * i + 2]),
                               __uint_as_float(v[4 * i + 3]));
        }
      }
    } else {
      // an empty row range contributes zeros
      for (int pp = 0; pp < p.pairs; ++pp) {
        const int t0 = pp * 2 < p.taps - 1 ? pp * 2 : p.taps - 2;
        const int tap = q < 2 ? t0 : t0 + 1;
        const int c = (q & 1) * 32 + lane;
        float* dst = p.partial + (((int64_t)item * p.taps + tap) * 64 + c) * 64;
        for (int i = 0; i < 64; ++i) dst[i] = 0.0f;
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

// dW[kbcb][tap][c][k] = sum over the Z partials of that block pair in a
// fixed order: kZS slices of consecutive partials (ascending z inside a
// slice, loads issued 8 at a time), then the slice sums in slice order.  A CTA
// owns 64 float4 outputs x kZS slices, so the ~22 MB of partials stream with
// every SM loading (one thread per output over all Z left 36 CTAs with a
// 148-long load-latency chain each: 25 us).
constexpr int kZS = 4;
__device__ __forceinline__ void add4(float4& a, const float4& v) {
  a.x = __fadd_rn(a.x, v.x); a.y = __fadd_rn(a.y, v.y);
  a.z = __fadd_rn(a.z, v.z); a.w = __fadd_rn(a.w, v.w);
}
__global__ void __launch_bounds__(64 * kZS) conv_dw_reduce(const float4* __restrict__ partial,
                                                           float4* __restrict__ dw, int Z, int64_t per4,
                                                           int64_t blocks) {
  __shared__ float4 slice_sum[kZS][64];
  const int lo = threadIdx.x & 63, sl = threadIdx.x >> 6;
  const int zs = (Z + kZS - 1) / kZS, z0 = sl * zs, z1 = min(Z, z0 + zs);
  for (int64_t e0 = (int64_t)blockIdx.x * 64; e0 < per4 * blocks; e0 += (int64_t)gridDim.x * 64) {
    const int64_t e = e0 + lo;
    const bool on = e < per4 * blocks;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (on && z0 < z1) {
      const int64_t b = e / per4, o = e % per4;
      const float4* src = partial + (b * Z) * per4 + o;
      acc = src[(int64_t)z0 * per4];
      int zz = z0 + 1;
      for (; zz + 8 <= z1; zz += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(src + (int64_t)(zz + u) * per4);
#pragma unroll
        for (int u = 0; u < 8; ++u) add4(acc, v[u]);
      }
      for (; zz < z1; ++zz) add4(acc, __ldg(src + (int64_t)zz * per4));
    }
    slice_sum[sl][lo] = acc;
    __syncthreads();
    if (sl == 0 && on) {
      float4 r = slice_sum[0][lo];
      for (int q = 1; q < kZS; ++q)
        if (q * zs < Z) add4(r, slice_sum[q][lo]);
      dw[e] = r;
    }
    __syncthreads();
  }
}

inline int splits(int Kb, int Cb) {
  const int z = num_sms() / (Kb * Cb);
  return z < 1 ? 1 : z;
}

}  // namespace cdw

int64_t conv_dw_workspace_bytes(int Kb, int Cb, int R, int S) {
  return (int64_t)Kb * Cb * cdw::splits(Kb, Cb) * R * S * 64 * 64 * 4;
}

int conv_backward_weights_tc(int N, int Cb, int Kb, int H, int W, int R, int S, int pad, const void* x,
                             const void* dout, float* dw, void* workspace, cudaStream_t stream) {
  using namespace cdw;
  TPP_REQUIRE(R <= kMaxR && 2 * pad == R - 1 && 2 * pad == S - 1, TPP_E_UNSUPPORTED,
              "conv backward-weights implements 'same' padding with R <= 3");
  TPP_REQUIRE(W + S - 1 <= 64, TPP_E_UNSUPPORTED, "conv backward-weights needs W + S - 1 <= 64");
  TPP_REQUIRE(R * S >= 2 && (R * S + 1) / 2 <= kMaxPairs, TPP_E_UNSUPPORTED, "conv backward-weights needs 2..16 taps");
  Params p{};
  p.N = N; p.H = H; p.W = W; p.R = R; p.S = S; p.pad = pad; p.Cb = Cb; p.Kb = Kb;
  p.Z = splits(Kb, Cb);
  p.taps = R * S;
  p.pairs = (p.taps + 1) / 2;
  p.partial = reinterpret_cast<float*>(workspace);
  CUtensorMap mx, md;
  {
    const uint64_t dims[5] = {64, (uint64_t)W, (uint64_t)H, (uint64_t)Cb, (uint64_t)N};
    const uint64_t str[4] = {128, (uint64_t)W * 128, (uint64_t)H * W * 128, (uint64_t)Cb * H * W * 128};
    const uint32_t box[5] = {64, 64, (uint32_t)R, 1, 1};
    int rc = make_tma_map_5d(&mx, x, dims, str, box, 128);
    if (rc) return rc;
  }
  {
    const uint64_t dims[5] = {64, (uint64_t)W, (uint64_t)H, (uint64_t)Kb, (uint64_t)N};
    const uint64_t str[4] = {128, (uint64_t)W * 128, (uint64_t)H * W * 128, (uint64_t)Kb * H * W * 128};
    const uint32_t box[5] = {64, 64, 1, 1, 1};
    int rc = make_tma_map_5d(&md, dout, dims, str, box, 128);
    if (rc) return rc;
  }
  const int smem = kStages * kStageBytes + (2 * kStages + 1) * 8 + 16 + 1024;
  const bool rs3 = R == 3 && S == 3;
  auto kern = rs3 ? conv_dw_kernel<1> : conv_dw_kernel<0>;
  {
    cudaError_t e = ensure_smem_attr((const void*)conv_dw_kernel<1>, smem);
    if (e == cudaSuccess) e = ensure_smem_attr((const void*)conv_dw_kernel<0>, smem);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(conv_dw_kernel)");
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(Kb * Cb * p.Z);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_allowed();
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mx, md, p);
  if (e != cudaSuccess) return cuda_status(e, "cudaLaunchKernelEx(conv_dw_kernel)");
  TPP_CUDA_LAUNCH_CHECK("conv_dw_kernel");
  const int64_t per4 = (int64_t)p.taps * 64 * 64 / 4, blocks = (int64_t)Kb * Cb;
  int64_t grid = (per4 * blocks + 63) / 64;
  if (grid > 4096) grid = 4096;
  conv_dw_reduce<<<(unsigned)grid, 64 * cdw::kZS, 0, stream>>>(reinterpret_cast<const float4*>(workspace),
                                                       reinterpret_cast<float4*>(dw), p.Z, per4, blocks);
  TPP_CUDA_LAUNCH_CHECK("conv_dw_reduce");
  return TPP_OK;
}

}  // namespace tpp

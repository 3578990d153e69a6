// K10: INT8 BRGEMM on tcgen05 tensor cores (kind::i8, INT32 accumulate).
//
// The reference's INT8 contraction (contraction.py:75-85, 184-189, 259-322)
// widens int8 to int32 and accumulates C = beta*C + sum_i A_i B_i in int32
// (numpy wrap-around).  Integer addition is associative, so unlike the float
// paths ANY summation order gives the reference's bits: the tensor cores,
// split-K over CTAs and int32 atomics are all exact.  This engine serves
// STRIDE batches with plain (column-major) A:
//
//   A_i (m, k) at a + i*stride_a + m + k*lda   -> MN-major operand
//   B_i (k, n) at b + i*stride_b + k + n*ldb   -> K-major operand
//   C   (m, n) at c + m + n*ldc (int32)
//
// Each operand is ONE 3-D TMA map (dims {M|K, K|N, count}); a pipeline stage
// is one (batch entry, 128-deep K block) pair: a 128(M) x 128(K) A box and a
// 128(K) x BN B box, both 128-byte swizzled, zero-filled past M/N/K (zeros add
// nothing to an integer sum).  Per stage 4 x tcgen05.mma (M=128, N=BN, K=32).
//
// Work unit = (128 x BN output tile, slice of the count*kblocks reduction).
// With one slice the epilogue applies beta and stores; with several (small C,
// long reductions) a beta pre-pass runs first and every slice red.add's its
// partial -- exact in two's complement.
//
// Roles (192 threads): warp 0 TMA producer, warp 1 TMEM alloc + MMA issue,
// warps 2-5 epilogue (warp w reads TMEM lanes 32*(w%4)...), accumulator
// double-buffered in TMEM so the epilogue of unit u overlaps unit u+1.

#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace tpp {

using namespace sm100;

namespace i8 {

constexpr int BM = 128;       // output rows per tile (UMMA M, TMEM lanes)
constexpr int BKB = 128;      // K bytes per stage (one 128-byte swizzle row)
constexpr int kThreads = 192;

template <int BN, int STAGES, int CG = 1>
struct Smem {
  static constexpr int A_BYTES = BM * BKB;         // 16 KB: 128 K-rows x 128 M bytes
  static constexpr int B_BYTES = (BN / CG) * BKB;  // this CTA's BN/CG N-rows x 128 K bytes
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int BAR_OFF = STAGES * STAGE;
  static constexpr int BYTES = BAR_OFF + 256 + 1024;  // + barriers, + 1024 alignment slack
};

struct Params {
  int m, n, kblocks;
  int64_t iters;        // count * kblocks
  int tiles_m, tiles_n, slices;   // tiles_m: row tiles (pairs of 128-row tiles for CTA pairs)
  int64_t units;
  int32_t* c;
  int64_t ldc;
  int beta_mode;        // 0: C = acc, 1: C = C + acc, 2: C = C*ibeta + acc, 3: red.add (pre-scaled)
  int32_t ibeta;
};

// tcgen05.mma kind::i8: signed x signed -> s32, warp-collective issue
__device__ __forceinline__ void umma_i8_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_i8_pair_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                  uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__host__ __device__ constexpr uint32_t idesc_s8_s32(int m, int n) {
  return (2u << 4)                      // D format S32
         | (1u << 7)                    // A signed 8-bit
         | (1u << 10)                   // B signed 8-bit
         | (1u << 15)                   // A MN-major
         | ((uint32_t)(n >> 3) << 17)   // N / 8
         | ((uint32_t)(m >> 4) << 24);  // M / 16
}

__device__ __forceinline__ void unit_coords(const Params& p, int64_t u, int& tm, int& tn, int64_t& it0,
                                            int64_t& it1) {
  const int64_t tile = u / p.slices;
  const int sl = (int)(u - tile * p.slices);
  tm = (int)(tile % p.tiles_m);
  tn = (int)(tile / p.tiles_m);
  const int64_t per = (p.iters + p.slices - 1) / p.slices;
  it0 = sl * per;
  it1 = it0 + per < p.iters ? it0 + per : p.iters;
}

// CG = 2: CTA pairs (cluster of 2, cta_group::2): a 256 x BN tile per pair;
// each CTA stages its own 128 A rows and half of B, the leader issues M=256
// MMAs and commits to both CTAs -- per-CTA shared-memory traffic per MAC
// drops by a third, which is what the BN=256 1-CTA form is bound by.
template <int BN, int STAGES, int CG>
__global__ void __launch_bounds__(kThreads, 1)
brgemm_i8_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                 const Params p) {
  using S = Smem<BN, STAGES, CG>;
  constexpr bool PAIR = CG == 2;
  extern __shared__ uint8_t raw_smem[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw_smem) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;  // warp-uniform (uniform-datapath MMA issue)
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int64_t cl0 = PAIR ? blockIdx.x >> 1 : blockIdx.x;
  const int64_t ncl = PAIR ? gridDim.x >> 1 : gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4 * CG);  // one elected arrive per epilogue warp (of both CTAs)
    }
    fence_mbar_init();
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_b);
  }
  if (warp == 1) {
    if (PAIR) tmem_alloc_pair(tmem_slot, S::TMEM_COLS);
    else tmem_alloc(tmem_slot, S::TMEM_COLS);
  }
  tc_fence_before();
  if (PAIR) cluster_sync();  // the peer's TMA and arrivals target the leader's barriers
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // uniform (MMA operand)

  if (warp == 0) {
    // ---- TMA producer ----
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full_cl = PAIR ? mapa_shared(smem_u32(full), 0) : 0;
      for (int64_t u = cl0; u < p.units; u += ncl) {
        int tm, tn;
        int64_t it0, it1;
        unit_coords(p, u, tm, tn, it0, it1);
        const int row0 = (tm * CG + (int)rank) * BM, col0 = tn * BN + (int)rank * (BN / CG);
        for (int64_t it = it0; it < it1; ++it) {
          const int i = (int)(it / p.kblocks), kb = (int)(it - (int64_t)i * p.kblocks);
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = sm + stage * S::STAGE;
          if (PAIR) {
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * S::STAGE);
            tma_load_5d_pair(sa, &map_a, full_cl + 8 * stage, row0, kb * BKB, i, 0, 0);
            tma_load_5d_pair(sa + S::A_BYTES, &map_b, full_cl + 8 * stage, kb * BKB, col0, i, 0, 0);
          } else {
            mbar_arrive_expect_tx(&full[stage], S::STAGE);
            tma_load_5d(sa, &map_a, &full[stage], row0, kb * BKB, i, 0, 0);
            tma_load_5d(sa + S::A_BYTES, &map_b, &full[stage], kb * BKB, col0, i, 0, 0);
          }
          if (++stage == STAGES) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (whole warp, elected lane issues; pairs: the leader) ----
    constexpr uint32_t idesc = idesc_s8_s32(BM * CG, BN);
    int stage = 0;
    uint32_t phase = 0;
    int buf = 0;
    uint32_t tphase = 0;
    for (int64_t u = cl0; u < p.units && leader; u += ncl) {
      int tm, tn;
      int64_t it0, it1;
      unit_coords(p, u, tm, tn, it0, it1);
      mbar_wait(&tempty[buf], tphase ^ 1);
      tc_fence_after();
      const uint32_t acc = tmem_base + buf * BN;
      for (int64_t it = it0; it < it1; ++it) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(sm + stage * S::STAGE);
        const uint32_t sb = sa + S::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < BKB / 32; ++kk) {
          // A: MN-major, 32 K-rows (4 swizzle atoms of 8 x 128 B) per MMA
          const uint64_t ad = sw128_mnmajor_desc(sa + kk * 32 * 128, 16384);
          // B: K-major, 32 bytes of K per MMA inside the 128-byte row
          const uint64_t bd = sw128_kmajor_desc(sb + kk * 32);
          if (PAIR) umma_i8_pair_warp(acc, ad, bd, idesc, (it > it0 || kk > 0) ? 1u : 0u);
          else umma_i8_warp(acc, ad, bd, idesc, (it > it0 || kk > 0) ? 1u : 0u);
        }
        if (PAIR) umma_commit_pair_warp(&empty[stage], 3);
        else umma_commit_warp(&empty[stage]);
        if (++stage == STAGES) stage = 0, phase ^= 1;
      }
      if (PAIR) umma_commit_pair_warp(&tfull[buf], 3);
      else umma_commit_warp(&tfull[buf]);
      if (++buf == 2) buf = 0, tphase ^= 1;
    }
  } else {
    // ---- epilogue: TMEM -> int32 C ----
    const int quarter = warp & 3;
    int buf = 0;
    uint32_t tphase = 0;
    const uint32_t tempty_leader = PAIR ? mapa_shared(smem_u32(tempty), 0) : 0;
    for (int64_t u = cl0; u < p.units; u += ncl) {
      int tm, tn;
      int64_t it0, it1;
      unit_coords(p, u, tm, tn, it0, it1);
      mbar_wait(&tfull[buf], tphase);
      tc_fence_after();
      const int row = (tm * CG + (int)rank) * BM + quarter * 32 + lane;
      const bool has = it1 > it0;  // an empty slice contributes nothing (accumulator untouched)
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) + buf * BN + c0, v);
        tmem_ld_wait();
        if (!has || row >= p.m) continue;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = tn * BN + c0 + j;
          if (col >= p.n) continue;
          int32_t* cp = p.c + row + (int64_t)col * p.ldc;
          if (p.beta_mode == 3) {
            asm volatile("red.global.add.s32 [%0], %1;" ::"l"(cp), "r"(v[j]) : "memory");
          } else if (p.beta_mode == 0) {
            *cp = (int32_t)v[j];
          } else if (p.beta_mode == 1) {
            *cp = (int32_t)((uint32_t)*cp + v[j]);
          } else {
            *cp = (int32_t)((uint32_t)*cp * (uint32_t)p.ibeta + v[j]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR && !leader) mbar_arrive_cluster(tempty_leader + 8 * buf);
        else mbar_arrive(&tempty[buf]);
      }
      if (++buf == 2) buf = 0, tphase ^= 1;
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync();  // neither CTA leaves while the pair still uses its smem / TMEM
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (PAIR) tmem_dealloc_pair(tmem_base, S::TMEM_COLS);
    else tmem_dealloc(tmem_base, S::TMEM_COLS);
  }
}

// beta pre-pass for the sliced (red.add) form: C = beta*C in int32
__global__ void beta_scale_kernel(int32_t* c, int m, int n, int64_t ldc, int mode, int32_t ibeta) {
  const int64_t total = (int64_t)m * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / m), i = (int)(e - (int64_t)j * m);
    int32_t* cp = c + i + (int64_t)j * ldc;
    if (mode == 0) *cp = 0;
    else *cp = (int32_t)((uint32_t)*cp * (uint32_t)ibeta);
  }
}

static int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <int BN, int STAGES, int CG>
static int launch_cfg(const CUtensorMap& ma, const CUtensorMap& mb, const Params& p, cudaStream_t s) {
  using S = Smem<BN, STAGES, CG>;
  static_assert(S::BYTES <= 227 * 1024, "shared memory budget");
  auto kern = brgemm_i8_kernel<BN, STAGES, CG>;
  static std::once_flag once;
  cudaError_t attr = cudaSuccess;
  static int max_clusters = 0;
  std::call_once(once, [&] {
    max_clusters = sm_count() / CG;
    if (CG > 1 && ensure_smem_attr((const void*)kern, S::BYTES) == cudaSuccess) {
      cudaLaunchConfig_t q{};
      q.gridDim = dim3(sm_count());
      q.blockDim = dim3(kThreads);
      q.dynamicSmemBytes = S::BYTES;
      cudaLaunchAttribute ca[1];
      ca[0].id = cudaLaunchAttributeClusterDimension;
      ca[0].val.clusterDim.x = CG; ca[0].val.clusterDim.y = 1; ca[0].val.clusterDim.z = 1;
      q.attrs = ca;
      q.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &q) == cudaSuccess && n > 0 && n < max_clusters) max_clusters = n;
      cudaGetLastError();
    }
  });
  attr = ensure_smem_attr((const void*)kern, S::BYTES);
  if (attr != cudaSuccess) return cuda_status(attr, "cudaFuncSetAttribute(brgemm_i8_kernel)");
  const int64_t clusters = p.units < max_clusters ? p.units : max_clusters;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(clusters * CG));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = S::BYTES;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = CG > 1 ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, p);
  if (e != cudaSuccess) return cuda_status(e, "cudaLaunchKernelEx(brgemm_i8_kernel)");
  TPP_CUDA_LAUNCH_CHECK("brgemm_i8_kernel");
  return TPP_OK;
}

}  // namespace i8

// 1 = not applicable (caller falls back to the ordered engine), else a TPP status
int brgemm_i8_stride_tc(int m, int n, int k, const int8_t* a, int64_t lda, const int8_t* b, int64_t ldb,
                        int64_t stride_a, int64_t stride_b, int64_t count, int32_t* c, int64_t ldc, double beta,
                        cudaStream_t s) {
  using namespace i8;
  const bool aligned = (reinterpret_cast<uintptr_t>(a) % 16) == 0 && (reinterpret_cast<uintptr_t>(b) % 16) == 0 &&
                       lda % 16 == 0 && ldb % 16 == 0 && (count <= 1 || (stride_a % 16 == 0 && stride_b % 16 == 0)) &&
                       stride_a >= 0 && stride_b >= 0;
  if (!aligned || count < 1) return 1;
  Params p{};
  p.m = m;
  p.n = n;
  p.kblocks = (k + BKB - 1) / BKB;
  p.iters = count * p.kblocks;
  const int tiles_m1 = (m + BM - 1) / BM;
  const int BN = n > 128 ? 256 : (n > 64 ? 128 : 64);
  p.tiles_n = (n + BN - 1) / BN;
  // CTA pairs for the wide tiles when there are row tiles to pair up
  static const int forced_cg = getenv("TPP_I8_CG") ? atoi(getenv("TPP_I8_CG")) : 0;
  const bool pair_wave = BN == 256 && (int64_t)(tiles_m1 / 2) * p.tiles_n >= sm_count() / 2;
  const int CG = tiles_m1 < 2 || forced_cg == 1 ? 1 : (pair_wave || forced_cg == 2 ? 2 : 1);
  p.tiles_m = (tiles_m1 + CG - 1) / CG;
  const int64_t tiles = (int64_t)p.tiles_m * p.tiles_n;
  // slice the reduction when the tiles alone leave SMs idle (>= 4 stages per slice)
  int64_t slices = 1;
  if (tiles < sm_count()) {
    slices = sm_count() / tiles;
    const int64_t max_slices = p.iters / 4 > 0 ? p.iters / 4 : 1;
    if (slices > max_slices) slices = max_slices;
  }
  p.slices = (int)slices;
  p.units = tiles * slices;
  p.c = c;
  p.ldc = ldc;
  const int32_t ibeta = (int32_t)beta;  // numpy int32(beta): truncation toward zero
  p.ibeta = ibeta;
  if (slices > 1) {
    if (beta != 1.0) {
      const int64_t total = (int64_t)m * n;
      int64_t blocks = (total + 255) / 256;
      if (blocks > sm_count() * 8) blocks = sm_count() * 8;
      beta_scale_kernel<<<(unsigned)blocks, 256, 0, s>>>(c, m, n, ldc, beta == 0.0 ? 0 : 2, ibeta);
      TPP_CUDA_LAUNCH_CHECK("beta_scale_kernel");
    }
    p.beta_mode = 3;
  } else {
    p.beta_mode = beta == 0.0 ? 0 : (beta == 1.0 ? 1 : 2);
  }
  // A: dims {M, K, count}, B: dims {K, N, count} (1-byte elements, innermost first)
  CUtensorMap ma, mb;
  const uint64_t da[5] = {(uint64_t)m, (uint64_t)k, (uint64_t)count, 1, 1};
  const uint64_t sa[4] = {(uint64_t)lda, (uint64_t)(count > 1 ? stride_a : (int64_t)lda * k), 16, 16};
  const uint32_t ba[5] = {BM, BKB, 1, 1, 1};
  const uint64_t db[5] = {(uint64_t)k, (uint64_t)n, (uint64_t)count, 1, 1};
  const uint64_t sb[4] = {(uint64_t)ldb, (uint64_t)(count > 1 ? stride_b : (int64_t)ldb * n), 16, 16};
  const uint32_t bb[5] = {BKB, (uint32_t)(BN / CG), 1, 1, 1};
  if ((sa[1] % 16) || (sb[1] % 16)) return 1;
  int rc = make_tma_map_5d_u8(&ma, a, da, sa, ba);
  if (rc) return rc;
  rc = make_tma_map_5d_u8(&mb, b, db, sb, bb);
  if (rc) return rc;
  if (CG == 2) {
    switch (BN) {
      case 256: return launch_cfg<256, 6, 2>(ma, mb, p, s);
      case 128: return launch_cfg<128, 8, 2>(ma, mb, p, s);
      default: return launch_cfg<64, 8, 2>(ma, mb, p, s);
    }
  }
  switch (BN) {
    case 256: return launch_cfg<256, 4, 1>(ma, mb, p, s);
    case 128: return launch_cfg<128, 6, 1>(ma, mb, p, s);
    default: return launch_cfg<64, 8, 1>(ma, mb, p, s);
  }
}

}  // namespace tpp

// K1: BRGEMM in the reference's exact per-element order (SIMT).
//
// contraction.py:261-322: for every C element
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

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"

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

// Shared-memory variant: a CTA owns a TM x TN tile of C (one element per
// thread) and stages the tile's A rows and B columns of a chunk of batch
// entries in shared memory, so the serial per-element chain reads operands
// at shared-memory latency instead of waiting on L2 every step.  Same order,
// same bits as brgemm_ordered_kernel.
constexpr int kOTM = 16, kOTN = 8;  // 128 C elements per CTA
// entry slots: kES threads per C element, each running the partial-sum chains
// of every kES-th batch entry (independent chains); slot 0 then adds the
// parts to the accumulator in entry order
constexpr int kES = 4;

template <typename TIn>
__device__ __forceinline__ const TIn* batch_a(const OrderedParams& p, int64_t inst, int64_t i) {
  if (p.mode == 0) return reinterpret_cast<const TIn*>(p.a) + inst * p.inst_a + i * p.stride_a;
  if (p.mode == 1) return reinterpret_cast<const TIn*>(p.a) + p.a_offs[i];
  return reinterpret_cast<const TIn*>(p.a_ptrs[i]);
}
template <typename TIn>
__device__ __forceinline__ const TIn* batch_b(const OrderedParams& p, int64_t inst, int64_t i) {
  if (p.mode == 0) return reinterpret_cast<const TIn*>(p.b) + inst * p.inst_b + i * p.stride_b;
  if (p.mode == 1) return reinterpret_cast<const TIn*>(p.b) + p.b_offs[i];
  return reinterpret_cast<const TIn*>(p.b_ptrs[i]);
}

template <typename TIn>
__device__ __forceinline__ void stage_elem(TIn* dst, const TIn* src) {
  if constexpr (sizeof(TIn) == 4 || sizeof(TIn) == 8) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "n"((int)sizeof(TIn))
                 : "memory");
  } else {
    *dst = __ldg(src);
  }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// KC: compile-time reduce length (64 = the paper's blocks; 0 = runtime p.k).
// fast: FP32, plain layouts, 16-byte aligned rows/columns, full tile ->
// 16-byte cp.async staging.
template <typename TIn, typename TAcc, int KC>
__global__ void __launch_bounds__(kOTM * kOTN * kES)
brgemm_ordered_smem_kernel(OrderedParams p, int nb, int fast, unsigned long long* dbg,
                           const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                           int use_tma) {
  using A = Arith<TAcc>;
  using W = Widen<TIn, TAcc>;
  const int K = KC ? KC : p.k;
  extern __shared__ __align__(128) unsigned char osm[];
  __shared__ uint64_t tma_bar;  // TMA staging: one box of A rows + one of B columns per chunk
  uint32_t tma_ph = 0;
  TIn* As = reinterpret_cast<TIn*>(osm);            // [nb][K][kOTM]  (rows contiguous)
  TIn* Bs = As + (size_t)nb * K * kOTM;             // [nb][kOTN][K]  (columns contiguous)
  // [nb][kOTM * kOTN] partial sums, 16-byte aligned after the B columns
  TAcc* Ps = reinterpret_cast<TAcc*>((reinterpret_cast<uintptr_t>(Bs + (size_t)nb * K * kOTN) + 15) & ~uintptr_t(15));
  const int tiles_m = (p.m + kOTM - 1) / kOTM;
  const int m0 = (blockIdx.x % tiles_m) * kOTM, n0 = (blockIdx.x / tiles_m) * kOTN;
  const int tid = threadIdx.x, es = tid / (kOTM * kOTN), etid = tid % (kOTM * kOTN);
  const int r = etid % kOTM, cidx = etid / kOTM;
  const int mi = m0 + r, ni = n0 + cidx;
  const bool live = mi < p.m && ni < p.n;
  constexpr int nthr = kOTM * kOTN * kES;
  auto gt = [] { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; };
  if (dbg && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) dbg[0] = gt();
  if (use_tma) {
    if (tid == 0) {
      sm100::mbar_init(&tma_bar, 1);
      sm100::fence_mbar_init();
      sm100::prefetch_tmap(&tma_a);
      sm100::prefetch_tmap(&tma_b);
    }
    __syncthreads();
  }
  for (int64_t inst = blockIdx.y; inst < p.instances; inst += gridDim.y) {
    TAcc* c = reinterpret_cast<TAcc*>(p.c) + inst * p.inst_c;
    TAcc acc = TAcc(0);
    if (live) {
      if (p.beta == 0.0) acc = TAcc(0);
      else if (p.beta == 1.0) acc = c[mi + (int64_t)ni * p.ldc];
      else acc = A::mul(c[mi + (int64_t)ni * p.ldc], A::beta(p.beta));
    }
    for (int64_t i0 = 0; i0 < p.count; i0 += nb) {
      const int cnt = (int)min((int64_t)nb, p.count - i0);
      __syncthreads();  // previous chunk fully consumed
      // stage the chunk's A rows [m0, m0+kOTM) and B columns [n0, n0+kOTN)
      if (use_tma) {
        // [nb][K][kOTM] A rows and [nb][kOTN][K] B columns, entries past
        // `count` zero-filled (never read)
        if (tid == 0) {
          sm100::mbar_arrive_expect_tx(&tma_bar, (uint32_t)(nb * K * (kOTM + kOTN) * (int)sizeof(TIn)));
          sm100::tma_load_5d(As, &tma_a, &tma_bar, 2 * m0, 0, (int)i0, (int)inst, 0);
          sm100::tma_load_5d(Bs, &tma_b, &tma_bar, 0, n0, (int)i0, (int)inst, 0);
        }
        sm100::mbar_wait(&tma_bar, tma_ph);
        tma_ph ^= 1u;
      }
      for (int bi = 0; bi < (use_tma ? 0 : cnt); ++bi) {
        const TIn* ab = batch_a<TIn>(p, inst, i0 + bi);
        const TIn* bb = batch_b<TIn>(p, inst, i0 + bi);
        TIn* as = As + (size_t)bi * K * kOTM;
        TIn* bs = Bs + (size_t)bi * K * kOTN;
        if (fast) {
          // 16-byte copies: A row segments (4 per k), B column segments (K/4 per column)
          for (int j = tid; j < K * (kOTM / 4); j += nthr) {
            const int kk = j / (kOTM / 4), q = j % (kOTM / 4);
            cp_async16(as + kk * kOTM + q * 4, ab + m0 + q * 4 + (int64_t)kk * p.lda);
          }
          for (int j = tid; j < kOTN * (K / 4); j += nthr) {
            const int cc = j / (K / 4), q = j % (K / 4);
            cp_async16(bs + cc * K + q * 4, bb + q * 4 + (int64_t)(n0 + cc) * p.ldb);
          }
        } else {
          const int rr = tid % kOTM, m = m0 + rr;
#pragma unroll 4
          for (int kk = tid / kOTM; kk < K; kk += nthr / kOTM) {
            TIn* dst = as + kk * kOTM + rr;
            if (m < p.m) {
              const TIn* src = p.vnni ? ab + (int64_t)(kk / p.alpha) * p.m * p.alpha + (int64_t)m * p.alpha + (kk % p.alpha)
                                      : ab + m + (int64_t)kk * p.lda;
              stage_elem(dst, src);
            } else {
              *dst = TIn(0);
            }
          }
#pragma unroll 4
          for (int e = tid; e < kOTN * K; e += nthr) {
            const int cc = e / K, kk = e - cc * K, n = n0 + cc;
            TIn* dst = bs + cc * K + kk;
            if (n < p.n) stage_elem(dst, bb + kk + (int64_t)n * p.ldb);
            else *dst = TIn(0);
          }
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
      if (dbg && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) dbg[1] = gt();
      // The per-entry partial sums are independent chains (part_i depends
      // only on entry i); only acc = acc + part_i is ordered across entries
      // (contraction.py:307-314).  Slot es runs entries es, es + kES, ...
      int bi = es;
      for (; bi < cnt; bi += kES) {
        const TIn* a = As + (size_t)bi * K * kOTM + r;
        const TIn* b = Bs + (size_t)bi * K * kOTN + cidx * K;
        TAcc part = TAcc(0);
        if (KC) {
          // the whole 64-long chain unrolled: every operand load is issued
          // ahead of the dependent adds
          TAcc av[KC > 0 ? KC : 1], bv[KC > 0 ? KC : 1];
#pragma unroll
          for (int kk = 0; kk < KC; ++kk) { av[kk] = W::w(a[kk * kOTM]); bv[kk] = W::w(b[kk]); }
#pragma unroll
          for (int kk = 0; kk < KC; ++kk) part = A::add(part, A::mul(av[kk], bv[kk]));
        } else {
#pragma unroll 8
          for (int kk = 0; kk < K; ++kk) part = A::add(part, A::mul(W::w(a[kk * kOTM]), W::w(b[kk])));
        }
        Ps[(size_t)bi * (kOTM * kOTN) + etid] = part;
      }
      __syncthreads();
      if (es == 0)
        for (int e = 0; e < cnt; ++e) acc = A::add(acc, Ps[(size_t)e * (kOTM * kOTN) + etid]);
    }
    if (live && es == 0) c[mi + (int64_t)ni * p.ldc] = acc;
    if (dbg && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) dbg[2] = gt();
  }
}

template <typename TIn, typename TAcc, int KC>
static int launch_smem_kc(const OrderedParams& p, cudaStream_t s, int nb, int fast, size_t smem) {
  // FP32 stride batches with box-sized extents: stage each chunk with two TMA
  // boxes (A rows: FP32 seen as BF16 pairs {2m, k, entry, instance}; B
  // columns {2k, n, entry, instance}) instead of 16-byte cp.async
  CUtensorMap ma{}, mb{};
  int use_tma = 0;
  // (a zero instance stride -- every instance shares that operand, as the FP32
  // fc_forward's inst_b = 0 -- has no TMA encoding: the cp.async path then
  // indexes inst * p.inst_x itself)
  static const bool no_tma = getenv("TPP_ORDERED_CPASYNC") != nullptr;  // experiments
  const bool inst_ok = p.instances == 1 || (p.inst_a > 0 && p.inst_b > 0);
  if (fast && sizeof(TIn) == 4 && p.k <= 128 && nb <= 256 && p.stride_a > 0 && p.stride_b > 0 && inst_ok &&
      p.instances <= 0x7fffffff && p.count <= 0x7fffffff && !no_tma) {
    const uint64_t da[5] = {2 * (uint64_t)p.m, (uint64_t)p.k, (uint64_t)p.count, (uint64_t)p.instances, 1};
    const uint64_t sa[4] = {(uint64_t)p.lda * 4, (uint64_t)p.stride_a * 4, (uint64_t)(p.inst_a ? p.inst_a * 4 : 16),
                            16};
    const uint32_t ba[5] = {2 * kOTM, (uint32_t)p.k, (uint32_t)nb, 1, 1};
    const uint64_t db[5] = {2 * (uint64_t)p.k, (uint64_t)p.n, (uint64_t)p.count, (uint64_t)p.instances, 1};
    const uint64_t sb[4] = {(uint64_t)p.ldb * 4, (uint64_t)p.stride_b * 4, (uint64_t)(p.inst_b ? p.inst_b * 4 : 16),
                            16};
    const uint32_t bb[5] = {2 * (uint32_t)p.k, kOTN, (uint32_t)nb, 1, 1};
    if (make_tma_map_5d(&ma, p.a, da, sa, ba, 0) == TPP_OK && make_tma_map_5d(&mb, p.b, db, sb, bb, 0) == TPP_OK)
      use_tma = 1;
  }
  {
    cudaError_t e = ensure_smem_attr((const void*)brgemm_ordered_smem_kernel<TIn, TAcc, KC>, 200 * 1024);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(brgemm_ordered_smem)");
  }
  const int tiles = ((p.m + kOTM - 1) / kOTM) * ((p.n + kOTN - 1) / kOTN);
  dim3 grid((unsigned)tiles, (unsigned)(p.instances < 65535 ? p.instances : 65535));
  smem += (size_t)nb * kOTM * kOTN * sizeof(TAcc) + 16;  // partial sums
  brgemm_ordered_smem_kernel<TIn, TAcc, KC><<<grid, kOTM * kOTN * kES, smem, s>>>(p, nb, fast, debug_timestamps(), ma, mb,
                                                                            use_tma);
  TPP_CUDA_LAUNCH_CHECK("brgemm_ordered_smem_kernel");
  return TPP_OK;
}

template <typename TIn, typename TAcc>
static int launch_smem_t(const OrderedParams& p, cudaStream_t s, int nb, size_t smem) {
  // 16-byte staging: FP32 plain layouts, whole tiles, every row / column
  // segment 16-byte aligned (stride batches only: offsets live on the device)
  const bool fast = sizeof(TIn) == 4 && std::is_same<TIn, TAcc>::value && !p.vnni && p.mode == 0 &&
                    p.m % kOTM == 0 && p.n % kOTN == 0 && p.k % 4 == 0 && p.lda % 4 == 0 && p.ldb % 4 == 0 &&
                    p.stride_a % 4 == 0 && p.stride_b % 4 == 0 && p.inst_a % 4 == 0 && p.inst_b % 4 == 0 &&
                    reinterpret_cast<uintptr_t>(p.a) % 16 == 0 && reinterpret_cast<uintptr_t>(p.b) % 16 == 0;
  if (p.k == 64) return launch_smem_kc<TIn, TAcc, 64>(p, s, nb, fast ? 1 : 0, smem);
  return launch_smem_kc<TIn, TAcc, 0>(p, s, nb, fast ? 1 : 0, smem);
}

template <typename TIn, typename TAcc>
static int launch_t(const OrderedParams& p, cudaStream_t s) {
  // staged variant: chunks of up to nb batch entries (<= 96 KB of operands)
  static const bool global_only = getenv("TPP_ORDERED_GLOBAL") != nullptr;  // experiments
  if (p.k > 0 && p.count > 0 && !global_only) {
    const size_t per = (size_t)p.k * (kOTM + kOTN) * sizeof(TIn);
    int64_t nb = (int64_t)(96 * 1024) / (int64_t)per;
    if (nb > p.count) nb = p.count;
    if (nb >= 1) return launch_smem_t<TIn, TAcc>(p, s, (int)nb, (size_t)nb * per);
  }
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

// zero-count batches only apply the beta rule (contraction.py:300-315)
// Narrow-and-long FP32 BRGEMMs (m, k <= 16, many columns): the dilated
// conv1d's shape (kernels.py:350-378: C = K = 15 channels, S = 51 taps,
// Q = 60000 positions).  One thread per C column owns all m accumulators (the
// m independent per-row chains are the ILP).  Per CTA of kColN columns:
//   * the A blocks of kColChunk entries are staged in shared memory as
//     [entry][k][16] (zero-padded rows), read back as float4 broadcasts;
//   * each entry's B window (kColN columns x k values, contiguous when
//     ldb == k) is staged by coalesced 4-byte cp.async into a [col][k|1]
//     tile (odd pitch: conflict-free column reads), kColStages entries ahead.
// Per element the order is the reference's: part = +0; part += a*b over k
// ascending; acc += part over entries ascending (separately rounded).
constexpr int kColM = 16, kColK = 16, kColN = 64, kColChunk = 8, kColStages = 4;
constexpr int kColRows = 8;  // rows per thread: m > 8 takes two row groups per column

template <int KC>  // KC = p.k (compile-time: the inner loop carries no bounds checks)
__global__ void __launch_bounds__(2 * kColN) brgemm_ordered_cols_kernel(OrderedParams p) {
  __shared__ __align__(16) float As[kColChunk][KC][kColM];
  __shared__ __align__(16) float Bs[kColStages][(kColN * (KC | 1) + 3) & ~3];
  constexpr int pitch = KC | 1;
  const int n0 = blockIdx.x * kColN, ncols = min(kColN, (int)(p.n - n0));
  const int t = threadIdx.x, nthr = blockDim.x;
  const int col = t % kColN, r0 = (t / kColN) * kColRows;  // row group: warp-uniform
  const bool live = col < ncols;
  float* c = reinterpret_cast<float*>(p.c);
  float acc[kColRows];
#pragma unroll
  for (int mm = 0; mm < kColRows; ++mm) {
    float v = 0.f;
    if (live && r0 + mm < p.m && p.beta != 0.0) {
      v = c[r0 + mm + (int64_t)(n0 + col) * p.ldc];
      if (p.beta != 1.0) v = __fmul_rn(v, (float)p.beta);
    }
    acc[mm] = v;
  }
  // Staging walk: element e = col * k + kk of the window, e = t, t + nthr, ...
  // advanced incrementally (no per-element division).
  const int tile_elems = ncols * p.k;
  const int col0 = t / p.k, kk0 = t - col0 * p.k;
  const int dcol = nthr / p.k, dkk = nthr - dcol * p.k;
  // Contiguous windows (ldb == k, k odd: the dilated conv's case) are copied
  // as-is -- [col][k] with an odd pitch is already conflict-free -- with
  // 16-byte cp.async when the window start is 16-byte aligned.
  const bool contig = p.ldb == KC && (KC & 1);
  auto stage_b = [&](int64_t entry, int slot) {
    if (entry < p.count && contig) {
      const float* win = batch_b<float>(p, 0, entry) + (int64_t)n0 * KC;
      float* dst = Bs[slot];
      if ((reinterpret_cast<uintptr_t>(win) & 15) == 0) {
        const int v4 = tile_elems >> 2;
        for (int e = t; e < v4; e += nthr) cp_async16(dst + 4 * e, win + 4 * e);
        for (int e = 4 * v4 + t; e < tile_elems; e += nthr) stage_elem<float>(dst + e, win + e);
      } else {
        for (int e = t; e < tile_elems; e += nthr) stage_elem<float>(dst + e, win + e);
      }
    } else if (entry < p.count) {
      const float* src = batch_b<float>(p, 0, entry) + (int64_t)n0 * p.ldb + (int64_t)col0 * p.ldb + kk0;
      float* dst = Bs[slot] + col0 * pitch + kk0;
      int kk = kk0;
      for (int e = t; e < tile_elems; e += nthr) {
        stage_elem<float>(dst, src);
        kk += dkk;
        src += (int64_t)dcol * p.ldb + dkk;
        dst += dcol * pitch + dkk;
        if (kk >= p.k) { kk -= p.k; src += p.ldb - p.k; dst += pitch - p.k; }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int st = 0; st < kColStages - 1; ++st) stage_b(st, st);
  for (int64_t i0 = 0; i0 < p.count; i0 += kColChunk) {
    const int cnt = (int)min((int64_t)kColChunk, p.count - i0);
    __syncthreads();  // previous chunk's A reads done
    for (int e = t; e < cnt * KC * kColM; e += nthr) {
      const int bi = e / (KC * kColM), kk = (e / kColM) % KC, mm = e % kColM;
      float v = 0.f;
      if (mm < p.m) v = batch_a<float>(p, 0, i0 + bi)[mm + (int64_t)kk * p.lda];
      As[bi][kk][mm] = v;
    }
    for (int bi = 0; bi < cnt; ++bi) {
      const int64_t i = i0 + bi;
      asm volatile("cp.async.wait_group %0;" ::"n"(kColStages - 2) : "memory");
      __syncthreads();  // entry i's B tile (and, at bi == 0, the A chunk) visible; slot of i-1 free
      stage_b(i + kColStages - 1, (int)((i + kColStages - 1) % kColStages));
      if (live) {
        const float* bs = Bs[i % kColStages] + col * pitch;
        float part[kColRows];
#pragma unroll
        for (int mm = 0; mm < kColRows; ++mm) part[mm] = 0.f;
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
          const float bv = bs[kk];
          const float4* ar = reinterpret_cast<const float4*>(&As[bi][kk][r0]);
#pragma unroll
          for (int q = 0; q < kColRows / 4; ++q) {
            const float4 av = ar[q];
            part[4 * q + 0] = __fadd_rn(part[4 * q + 0], __fmul_rn(av.x, bv));
            part[4 * q + 1] = __fadd_rn(part[4 * q + 1], __fmul_rn(av.y, bv));
            part[4 * q + 2] = __fadd_rn(part[4 * q + 2], __fmul_rn(av.z, bv));
            part[4 * q + 3] = __fadd_rn(part[4 * q + 3], __fmul_rn(av.w, bv));
          }
        }
#pragma unroll
        for (int mm = 0; mm < kColRows; ++mm) acc[mm] = __fadd_rn(acc[mm], part[mm]);
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (live) {
#pragma unroll
    for (int mm = 0; mm < kColRows; ++mm)
      if (r0 + mm < p.m) c[r0 + mm + (int64_t)(n0 + col) * p.ldc] = acc[mm];
  }
}

// Sliding-window variant: STRIDE batches whose B blocks are column windows
// of one contiguous matrix (ldb == k, stride_b = sh columns) -- the dilated
// conv's taps, entry s reading input columns q + s*d.  A CTA covers ncb
// columns; the union of its windows (ncb + (count-1)*sh columns) and every
// entry's A block are staged ONCE (cp.async), then the entry loop is pure
// shared-memory reads + arithmetic with no barrier.  One CTA per SM with the
// columns split evenly (ncb = n / #SMs rounded up to a warp), so the single
// wave is balanced.  Same per-element order as the kernels above.
template <int KC>
__global__ void __launch_bounds__(512, 1) brgemm_ordered_window_kernel(OrderedParams p, int ncb, int sh) {
  extern __shared__ __align__(16) float wsm[];
  float* As = wsm;                                   // [count][KC][16], rows >= m zero
  float* Bu = wsm + (size_t)p.count * KC * kColM;    // [U][KC] window union
  const int n0 = blockIdx.x * ncb, ncols = min(ncb, (int)(p.n - n0));
  if (ncols <= 0) return;
  const int t = threadIdx.x, nthr = blockDim.x;
  const int ucols = ncols + (int)(p.count - 1) * sh;
  {
    const float* win = reinterpret_cast<const float*>(p.b) + (int64_t)n0 * KC;
    const int elems = ucols * KC;
    int done = 0;
    if ((reinterpret_cast<uintptr_t>(win) & 15) == 0) {
      done = elems & ~3;
      for (int e = 4 * t; e < done; e += 4 * nthr) cp_async16(Bu + e, win + e);
    }
    for (int e = done + t; e < elems; e += nthr) stage_elem<float>(Bu + e, win + e);
    asm volatile("cp.async.commit_group;" ::: "memory");
    const float* a = reinterpret_cast<const float*>(p.a);
    for (int e = t; e < (int)p.count * KC * kColM; e += nthr) {
      const int mm = e % kColM, kk = (e / kColM) % KC, bi = e / (KC * kColM);
      As[e] = mm < p.m ? a[(int64_t)bi * p.stride_a + mm + (int64_t)kk * p.lda] : 0.f;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
  }
  // Thread -> (row group, columns col and col + ncb/2): every A broadcast
  // feeds two columns' products.  (A warp straddling two row groups reads two
  // A addresses per LDS -- harmless.)
  const int half = ncb / 2;
  const int g = t / half, col = t - g * half;
  const int r0 = g * kColRows;
  if (col >= ncols) return;
  const bool two = col + half < ncols;
  float* c0 = reinterpret_cast<float*>(p.c) + (int64_t)(n0 + col) * p.ldc + r0;
  float* c1 = c0 + (int64_t)half * p.ldc;
  float acc0[kColRows], acc1[kColRows];
#pragma unroll
  for (int mm = 0; mm < kColRows; ++mm) {
    float v0 = 0.f, v1 = 0.f;
    if (r0 + mm < p.m && p.beta != 0.0) {
      v0 = c0[mm];
      if (two) v1 = c1[mm];
      if (p.beta != 1.0) v0 = __fmul_rn(v0, (float)p.beta), v1 = __fmul_rn(v1, (float)p.beta);
    }
    acc0[mm] = v0;
    acc1[mm] = v1;
  }
  const float* bs = Bu + col * KC;  // column col + half is half * KC further (inside the union)
  const float* as = As + r0;
  for (int i = 0; i < (int)p.count; ++i, bs += sh * KC, as += KC * kColM) {
    float part0[kColRows], part1[kColRows];
#pragma unroll
    for (int mm = 0; mm < kColRows; ++mm) part0[mm] = 0.f, part1[mm] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      const float b0 = bs[kk], b1 = bs[half * KC + kk];
      const float4* ar = reinterpret_cast<const float4*>(as + kk * kColM);
#pragma unroll
      for (int q = 0; q < kColRows / 4; ++q) {
        const float4 av = ar[q];
        part0[4 * q + 0] = __fadd_rn(part0[4 * q + 0], __fmul_rn(av.x, b0));
        part0[4 * q + 1] = __fadd_rn(part0[4 * q + 1], __fmul_rn(av.y, b0));
        part0[4 * q + 2] = __fadd_rn(part0[4 * q + 2], __fmul_rn(av.z, b0));
        part0[4 * q + 3] = __fadd_rn(part0[4 * q + 3], __fmul_rn(av.w, b0));
        part1[4 * q + 0] = __fadd_rn(part1[4 * q + 0], __fmul_rn(av.x, b1));
        part1[4 * q + 1] = __fadd_rn(part1[4 * q + 1], __fmul_rn(av.y, b1));
        part1[4 * q + 2] = __fadd_rn(part1[4 * q + 2], __fmul_rn(av.z, b1));
        part1[4 * q + 3] = __fadd_rn(part1[4 * q + 3], __fmul_rn(av.w, b1));
      }
    }
#pragma unroll
    for (int mm = 0; mm < kColRows; ++mm) {
      acc0[mm] = __fadd_rn(acc0[mm], part0[mm]);
      acc1[mm] = __fadd_rn(acc1[mm], part1[mm]);
    }
  }
#pragma unroll
  for (int mm = 0; mm < kColRows; ++mm) {
    if (r0 + mm < p.m) {
      c0[mm] = acc0[mm];
      if (two) c1[mm] = acc1[mm];
    }
  }
}

// Window-path plan: 0 = not applicable, else fills ncb / sh / smem bytes.
static bool window_plan(const OrderedParams& p, int* ncb, int* sh, int* smem) {
  if (p.mode != 0 || (p.k & 1) == 0 || p.ldb != p.k || p.stride_b < 0 || p.stride_b % p.k != 0) return false;
  const int64_t groups = (p.m + kColRows - 1) / kColRows;
  int64_t cols = (p.n + num_sms() - 1) / num_sms();
  cols = (cols + 1) & ~int64_t(1);
  cols = std::min<int64_t>(cols, 512 / groups * 2);  // threads = groups * cols / 2 <= 512
  const int64_t shift = p.stride_b / p.k;
  // (the last CTA's threads whose second column lies past n still read --
  // and ignore -- union slots up to column cols - 1 + (count - 1) * shift)
  const int64_t bytes = p.count * p.k * kColM * 4 + (cols + (p.count - 1) * shift) * p.k * 4;
  if (bytes > 200 * 1024 || shift > (1 << 20)) return false;
  *ncb = (int)cols;
  *sh = (int)shift;
  *smem = (int)bytes;
  return true;
}

int launch_brgemm_ordered(const OrderedParams& p, int in_dtype, cudaStream_t s) {
  if (p.m == 0 || p.n == 0 || p.instances == 0) return TPP_OK;
  static const bool no_cols = getenv("TPP_ORDERED_NO_COLS") != nullptr;  // experiments
  if (in_dtype == TPP_FP32 && !p.vnni && p.instances == 1 && p.m <= kColM && p.k >= 1 && p.k <= kColK && p.n >= 2048 &&
      p.count > 0 && !no_cols) {
    static const bool no_window = getenv("TPP_ORDERED_NO_WINDOW") != nullptr;  // experiments
    int ncb = 0, sh = 0, smem = 0;
    if (!no_window && window_plan(p, &ncb, &sh, &smem)) {
      const int wthreads = ncb / 2 * ((p.m + kColRows - 1) / kColRows);
      const int wblocks = (int)((p.n + ncb - 1) / ncb);
      switch (p.k) {
#define TPP_WIN_K(K)                                                                                  \
  case K:                                                                                             \
    if (ensure_smem_attr((const void*)brgemm_ordered_window_kernel<K>, smem) != cudaSuccess) break;  \
    brgemm_ordered_window_kernel<K><<<wblocks, wthreads, smem, s>>>(p, ncb, sh);                       \
    TPP_CUDA_LAUNCH_CHECK("brgemm_ordered_window_kernel");                                             \
    return TPP_OK;
        TPP_WIN_K(1) TPP_WIN_K(3) TPP_WIN_K(5) TPP_WIN_K(7) TPP_WIN_K(9) TPP_WIN_K(11) TPP_WIN_K(13) TPP_WIN_K(15)
#undef TPP_WIN_K
      }
    }
    const int blocks = (int)((p.n + kColN - 1) / kColN);
    const int threads = kColN * ((p.m + kColRows - 1) / kColRows);
    switch (p.k) {
#define TPP_COLS_K(K) case K: brgemm_ordered_cols_kernel<K><<<blocks, threads, 0, s>>>(p); break;
      TPP_COLS_K(1) TPP_COLS_K(2) TPP_COLS_K(3) TPP_COLS_K(4) TPP_COLS_K(5) TPP_COLS_K(6) TPP_COLS_K(7)
      TPP_COLS_K(8) TPP_COLS_K(9) TPP_COLS_K(10) TPP_COLS_K(11) TPP_COLS_K(12) TPP_COLS_K(13)
      TPP_COLS_K(14) TPP_COLS_K(15) TPP_COLS_K(16)
#undef TPP_COLS_K
    }
    TPP_CUDA_LAUNCH_CHECK("brgemm_ordered_cols_kernel");
    return TPP_OK;
  }
  switch (in_dtype) {
    case TPP_FP32: return launch_t<float, float>(p, s);
    case TPP_FP64: return launch_t<double, double>(p, s);
    case TPP_BF16: return launch_t<uint16_t, float>(p, s);
    case TPP_INT8: return launch_t<int8_t, int32_t>(p, s);
    default: return fail(TPP_E_TENSOR, "unsupported BRGEMM input dtype");
  }
}

}  // namespace tpp

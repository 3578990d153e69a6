// K4 / K9: LayerNorm equation TPP, softmax, split-SGD — bitwise to the reference.
//
// LayerNorm (kernels.py:134-176): per row, FP32 sums of x and x*x folded in
// ascending column order (ops.py:484-522), float64 glue
//     mu = s/n ; var = ss/n - mu*mu ; rstd = 1/sqrt(var + eps)
// stored as FP32 scale = rstd, shift = -mu*rstd, then the scaling equation of
// two cascaded MULADDs  out = B + (shift + x*scale) * G  (ops.py:812-815).
// The reference order is one sequential chain per row, so one thread owns a
// row's statistics; what makes it fast on B200 is that the chain reads come
// from a coalesced access pattern (column-major view: consecutive threads =
// consecutive rows) or from shared memory (blocked layout), never from
// scattered HBM.

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace tpp {

__device__ __forceinline__ float nload(const DView& v, int i, int j) {
  const int pi = (v.bcast == TPP_BCAST_ROW || v.bcast == TPP_BCAST_SCALAR) ? 0 : i;
  const int pj = (v.bcast == TPP_BCAST_COL || v.bcast == TPP_BCAST_SCALAR) ? 0 : j;
  const int64_t idx = pi + (int64_t)pj * v.ld;
  if (v.dtype == TPP_BF16) return bf16_to_f32(reinterpret_cast<const uint16_t*>(v.p)[idx]);
  return reinterpret_cast<const float*>(v.p)[idx];
}

__device__ __forceinline__ void row_glue(float s, float ss, int n, double eps, float& scale,
                                         float& shift, double& mu, double& var) {
  mu = (double)s / (double)n;
  var = __dsub_rn((double)ss / (double)n, __dmul_rn(mu, mu));
  const double rstd = 1.0 / sqrt(__dadd_rn(var, eps));
  scale = (float)rstd;
  shift = (float)__dmul_rn(-mu, rstd);
}

// ---- column-major view: one thread per row, coalesced across threads -------
__global__ void layernorm_view_kernel(DView x, DView g, DView b, double eps, void* out, int out_ld,
                                      int out_dtype, float* mean_out, float* var_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= x.rows) return;
  const int n = x.cols;
  float s = 0.0f, ss = 0.0f;
  for (int j = 0; j < n; ++j) {
    const float v = nload(x, i, j);
    s = __fadd_rn(s, v);
    ss = __fadd_rn(ss, __fmul_rn(v, v));
  }
  float scale, shift;
  double mu, var;
  row_glue(s, ss, n, eps, scale, shift, mu, var);
  if (mean_out) mean_out[i] = (float)mu;
  if (var_out) var_out[i] = (float)var;
  for (int j = 0; j < n; ++j) {
    const float v = nload(x, i, j);
    const float inner = __fadd_rn(shift, __fmul_rn(v, scale));
    const float r = __fadd_rn(nload(b, i, j), __fmul_rn(inner, nload(g, i, j)));
    const int64_t o = i + (int64_t)j * out_ld;
    if (out_dtype == TPP_BF16) reinterpret_cast<uint16_t*>(out)[o] = f32_to_bf16(r);
    else reinterpret_cast<float*>(out)[o] = r;
  }
}

int launch_layernorm_view(const DView& x, const DView& g, const DView& b, double eps, void* out,
                          int out_ld, int out_dtype, float* mean_out, float* var_out,
                          cudaStream_t s) {
  if (x.rows == 0) return TPP_OK;
  const int threads = 128;
  layernorm_view_kernel<<<(x.rows + threads - 1) / threads, threads, 0, s>>>(
      x, g, b, eps, out, out_ld, out_dtype, mean_out, var_out);
  TPP_CUDA_LAUNCH_CHECK("layernorm_view_kernel");
  return TPP_OK;
}

// ---- blocked activations [n_b][m_b][bn][bm] (tokens x features) -------------
// CTA = 32 tokens of one token block, all F = m_b*bm features staged in smem
// (row pitch F+2 elements: conflict-free per-thread row walks).  Phase 1:
// coalesced HBM -> smem.  Phase 2: thread t walks its token's features
// ascending (the reference fold).  Phase 3: all threads apply the scaling
// equation and store coalesced.
template <typename T>
__global__ void __launch_bounds__(256)
layernorm_blocked_kernel(int n_b, int m_b, int bn, int bm, const T* __restrict__ x,
                         const float* __restrict__ gamma, const float* __restrict__ beta,
                         double eps, T* __restrict__ out, float* mean_out, float* var_out) {
  extern __shared__ __align__(16) uint8_t lsm[];
  const int F = m_b * bm;
  const int pitch = F + (sizeof(T) == 2 ? 2 : 1);
  T* rows = reinterpret_cast<T*>(lsm);
  float* sc = reinterpret_cast<float*>(lsm + (((size_t)32 * pitch * sizeof(T) + 15) & ~(size_t)15));
  float* sh = sc + 32;
  const int chunks_per_blk = (bn + 31) / 32;
  const int nb = blockIdx.x / chunks_per_blk;
  const int n0 = (blockIdx.x % chunks_per_blk) * 32;
  const int T_ = min(32, bn - n0);
  // phase 1
  for (int mb = 0; mb < m_b; ++mb) {
    const T* src = x + (((int64_t)nb * m_b + mb) * bn + n0) * bm;
    for (int e = threadIdx.x; e < T_ * bm; e += blockDim.x) {
      const int t = e / bm, m = e % bm;
      rows[t * pitch + mb * bm + m] = src[e];
    }
  }
  __syncthreads();
  // phase 2
  if (threadIdx.x < T_) {
    const T* r = rows + threadIdx.x * pitch;
    float s = 0.0f, ss = 0.0f;
    for (int f = 0; f < F; ++f) {
      float v;
      if (sizeof(T) == 2) v = bf16_to_f32(reinterpret_cast<const uint16_t*>(r)[f]);
      else v = reinterpret_cast<const float*>(r)[f];
      s = __fadd_rn(s, v);
      ss = __fadd_rn(ss, __fmul_rn(v, v));
    }
    float scale, shift;
    double mu, var;
    row_glue(s, ss, F, eps, scale, shift, mu, var);
    sc[threadIdx.x] = scale;
    sh[threadIdx.x] = shift;
    const int64_t tok = (int64_t)nb * bn + n0 + threadIdx.x;
    if (mean_out) mean_out[tok] = (float)mu;
    if (var_out) var_out[tok] = (float)var;
  }
  __syncthreads();
  // phase 3
  for (int mb = 0; mb < m_b; ++mb) {
    T* dst = out + (((int64_t)nb * m_b + mb) * bn + n0) * bm;
    for (int e = threadIdx.x; e < T_ * bm; e += blockDim.x) {
      const int t = e / bm, m = e % bm;
      const int f = mb * bm + m;
      float v;
      if (sizeof(T) == 2) v = bf16_to_f32(reinterpret_cast<const uint16_t*>(rows)[t * pitch + f]);
      else v = reinterpret_cast<const float*>(rows)[t * pitch + f];
      const float inner = __fadd_rn(sh[t], __fmul_rn(v, sc[t]));
      const float gv = gamma ? gamma[f] : 1.0f;
      const float bv = beta ? beta[f] : 0.0f;
      const float res = __fadd_rn(bv, __fmul_rn(inner, gv));
      if (sizeof(T) == 2) reinterpret_cast<uint16_t*>(dst)[e] = f32_to_bf16(res);
      else reinterpret_cast<float*>(dst)[e] = res;
    }
  }
}

// ---- blocked BF16, bm == 64, bn % 32 == 0: smem-transposed, vectorised ------
// CTA = 32 tokens of one token block.  (1) all 128 threads stream the 32
// tokens' 16 x 4 KB feature blocks into smem with coalesced 16-byte loads;
// (2) warp 0 folds each token's row in the reference's ascending order with
// LDS.128 (rows padded by 16 B: conflict-free); (3) all threads apply the
// scaling equation and store coalesced 16-byte chunks.
__device__ __forceinline__ void fold8(const uint4& v, float& s, float& ss) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float a = __uint_as_float(w[e] << 16), b = __uint_as_float(w[e] & 0xFFFF0000u);
    s = __fadd_rn(s, a);
    ss = __fadd_rn(ss, __fmul_rn(a, a));
    s = __fadd_rn(s, b);
    ss = __fadd_rn(ss, __fmul_rn(b, b));
  }
}

__global__ void __launch_bounds__(256)
layernorm_blocked_bf16_v(int n_b, int m_b, int bn, const uint4* __restrict__ x,
                         const float4* __restrict__ gamma, const float4* __restrict__ beta, double eps,
                         uint4* __restrict__ out, float* mean_out, float* var_out) {
  extern __shared__ __align__(16) uint4 lv[];
  const int F8 = m_b * 8;              // uint4 per token row
  const int pitch = F8 + 1;            // +16 B: LDS.128 across rows conflict-free
  float* sc = reinterpret_cast<float*>(lv + 32 * pitch);
  float* sh = sc + 32;
  const int chunks = bn / 32;
  const int nb = blockIdx.x / chunks;
  const int n0 = (blockIdx.x - nb * chunks) * 32;
  // block mb of these 32 tokens is 32 x 8 uint4 contiguous: one uint4 per thread
  const int tid = threadIdx.x, t = tid >> 3, c = tid & 7;
  const uint4* src = x + ((int64_t)nb * m_b * bn + n0) * 8 + tid;
  uint4* dst = out + ((int64_t)nb * m_b * bn + n0) * 8 + tid;
  const int64_t bstep = (int64_t)bn * 8;
  uint4* mine = lv + t * pitch + c;
  // (1) 8 independent loads in flight per thread
  for (int mb0 = 0; mb0 < m_b; mb0 += 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (mb0 + u < m_b) v[u] = __ldg(src + (mb0 + u) * bstep);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (mb0 + u < m_b) mine[(mb0 + u) * 8] = v[u];
  }
  __syncthreads();
  // (2) the reference fold, one thread per token
  if (tid < 32) {
    const uint4* row = lv + tid * pitch;
    float s = 0.0f, ss = 0.0f;
#pragma unroll 8
    for (int k = 0; k < F8; ++k) fold8(row[k], s, ss);
    float scale, shift;
    double mu, var;
    row_glue(s, ss, m_b * 64, eps, scale, shift, mu, var);
    sc[tid] = scale;
    sh[tid] = shift;
    const int64_t tok = (int64_t)nb * bn + n0 + tid;
    if (mean_out) mean_out[tok] = (float)mu;
    if (var_out) var_out[tok] = (float)var;
  }
  __syncthreads();
  // (3) out = B + (shift + x*scale)*G, 8 features per thread per block
  const float scl = sc[t], shf = sh[t];
  for (int mb = 0; mb < m_b; ++mb) {
    const uint4 v = mine[mb * 8];
    float g[8], b[8];
    if (gamma) {
      const float4 g0 = __ldg(gamma + mb * 16 + c * 2), g1 = __ldg(gamma + mb * 16 + c * 2 + 1);
      g[0] = g0.x; g[1] = g0.y; g[2] = g0.z; g[3] = g0.w; g[4] = g1.x; g[5] = g1.y; g[6] = g1.z; g[7] = g1.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) g[i] = 1.0f;
    }
    if (beta) {
      const float4 b0 = __ldg(beta + mb * 16 + c * 2), b1 = __ldg(beta + mb * 16 + c * 2 + 1);
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w; b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) b[i] = 0.0f;
    }
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float a0 = __uint_as_float(w[q] << 16), a1 = __uint_as_float(w[q] & 0xFFFF0000u);
      const float r0 = __fadd_rn(b[2 * q], __fmul_rn(__fadd_rn(shf, __fmul_rn(a0, scl)), g[2 * q]));
      const float r1 = __fadd_rn(b[2 * q + 1], __fmul_rn(__fadd_rn(shf, __fmul_rn(a1, scl)), g[2 * q + 1]));
      o[q] = pack2_bf16_ref(r0, r1);
    }
    dst[mb * bstep] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// ---- persistent TMA pipeline for BF16 blocked LayerNorm ---------------------
// One CTA per SM walks groups of 16 tokens.  A group (16 tokens x F features,
// F = m_b * 64) is ONE 5-D TMA box (128B-swizzled: lane t reading its row's
// 16-byte chunk c at c ^ (t & 7) is bank-conflict free) into a ring of
// `stages` buffers.  Warp roles:
//   warp 0        TMA loads (ring ahead) and TMA stores of finished groups
//   warps 1..4    the reference fold: one lane per token, FP32 ascending sums
//                 of x and x*x, float64 glue -> (scale, shift)
//   warps 5..12   the scaling equation in place (16 B per thread per step),
//                 then the group leaves through a TMA store from the same buffer
// so HBM reads, the latency-bound folds and the writes of different groups
// overlap; 16 x F x 2 bytes cross HBM once in each direction.
// waits sleep on the barrier (spin = 1: plain try_wait loop, for profiling tools)
#define LN_WAIT(bar, par) ((spin & 1) ? mbar_wait((bar), (par)) : mbar_wait_sleep((bar), (par)))
namespace lnt {
constexpr int kTok = 16;
constexpr int kFoldWarps = 4;
constexpr int kApplyWarps = 16;
constexpr int kApplyTeams = 4;    // teams apply different groups concurrently
constexpr int kTeamWarps = kApplyWarps / kApplyTeams;
constexpr int kApplySlabs = kTeamWarps * 32 / (kTok * 8);  // slabs a team covers per pass
constexpr int kThreads = 32 * (1 + kFoldWarps + kApplyWarps);
constexpr int kMaxStages = 8;
constexpr int kRingBytes = 224 * 1024;  // 7 groups of 16 x 1024 bf16: a CTA's whole share of cfg 3
}  // namespace lnt

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, const uint4& v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// FAST = 1: the tolerance mode (tree order allowed within
// 1e-5): per token 8 interleaved partial sums (chain 8x shorter) with fused
// x*x, and the scaling equation as two FMAs on element pairs.  FAST = 0 is
// the bitwise reference order.
template <int FAST>
__global__ void __launch_bounds__(lnt::kThreads, 1)
layernorm_blocked_tma(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_o,
                      int n_groups, int bn, int m_b, int stages, const float* __restrict__ gamma,
                      const float* __restrict__ beta, double eps, float* mean_out, float* var_out, int spin,
                      unsigned long long* dbg) {
  using namespace sm100;
  using namespace lnt;
  extern __shared__ __align__(1024) uint8_t ln_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ln_raw) + 1023) & ~uintptr_t(1023));
  const int gbytes = kTok * m_b * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * gbytes);
  uint64_t* stat = full + kMaxStages;
  uint64_t* done = stat + kMaxStages;
  float2* st = reinterpret_cast<float2*>(done + kMaxStages);  // [stage][token] (scale, shift)
  // seq[s] = group whose load was last issued into buffer s: a fold warp may
  // run ahead of buffer reuse, and an mbarrier parity wait cannot tell phase
  // u from phase u-2, so it first waits for its group's load to be issued
  volatile int* seq = reinterpret_cast<volatile int*>(st + kMaxStages * kTok);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    prefetch_tmap(&map_x);
    prefetch_tmap(&map_o);
    for (int s = 0; s < stages; ++s) {
      seq[s] = -1;
      mbar_init(&full[s], 1);
      mbar_init(&stat[s], 1);
      mbar_init(&done[s], kTeamWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const unsigned long long t_resident = dbg ? globaltimer_ns() : 0;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (dbg && threadIdx.x == 0) dbg[500 + blockIdx.x % 64] = t_resident;
  const int my = (n_groups - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const uint32_t sbase = smem_u32(sm);
  if (dbg && blockIdx.x == 0 && threadIdx.x == 0) dbg[0] = globaltimer_ns();
  if (dbg && threadIdx.x == 0) dbg[200 + 2 * blockIdx.x] = globaltimer_ns();

  if (warp == 0) {
    if (lane == 0) {
      int nl = 0, ns = 0;
      while (ns < my) {
        while (nl < my && nl < ns + stages) {
          const int s = nl % stages;
          if (nl >= stages) bulk_wait_read<0>();  // the store of group nl - stages has left buffer s
          const int t0 = ((int)blockIdx.x + nl * (int)gridDim.x) * kTok;
          seq[s] = nl;
          mbar_arrive_expect_tx(&full[s], gbytes);
          tma_load_5d(sm + s * gbytes, &map_x, &full[s], 0, t0 % bn, 0, t0 / bn, 0);
          if (dbg && blockIdx.x == 0 && (nl) < 16) dbg[8 + 5 * (nl) + 0] = globaltimer_ns();
          ++nl;
        }
        const int s = ns % stages;
        LN_WAIT(&done[s], (ns / stages) & 1);
        const int t0 = ((int)blockIdx.x + ns * (int)gridDim.x) * kTok;
        tma_store_5d(&map_o, sm + s * gbytes, 0, t0 % bn, 0, t0 / bn, 0);
        bulk_commit();
        if (dbg && blockIdx.x == 0 && (ns) < 16) dbg[8 + 5 * (ns) + 4] = globaltimer_ns();
        ++ns;
      }
      bulk_wait_read<0>();  // smem outlives the stores' reads; the writes complete with the grid
      if (dbg) dbg[201 + 2 * blockIdx.x] = globaltimer_ns();
    }
  } else if (warp <= kFoldWarps) {
    // a fold warp takes two groups at once: lanes 0-15 group 2P, 16-31 group 2P+1
    const int half = lane >> 4, t = lane & (kTok - 1);
    for (int P = warp - 1; 2 * P < my; P += kFoldWarps) {
      const int i = 2 * P + half;
      const bool live = i < my;
      const int s = (live ? i : 2 * P) % stages;
      for (int g = 2 * P; g < 2 * P + 2 && g < my; ++g) {
        while (seq[g % stages] != g) __nanosleep(64);
        LN_WAIT(&full[g % stages], (g / stages) & 1);
      }
      if (lane == 0) { if (dbg && blockIdx.x == 0 && (2 * P) < 16) dbg[8 + 5 * (2 * P) + 1] = globaltimer_ns(); }
      const uint32_t row = sbase + s * gbytes + t * 128;
      const int sw = t & 7;
      float a = 0.0f, b = 0.0f;
      float pa[8], pb[8];  // FAST: one partial pair per chunk slot
#pragma unroll
      for (int c = 0; c < 8; ++c) { pa[c] = 0.0f; pb[c] = 0.0f; }
      // software pipeline: the next slab's 8 chunks are in flight while this
      // slab is folded (the fold itself is a 2 x F-long FADD chain per token)
      uint4 cur[8], nxt[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) cur[c] = lds128(row + ((c ^ sw) << 4));
      for (int cb = 0; cb < m_b; ++cb) {
        const uint32_t nrow = row + (cb + 1 < m_b ? cb + 1 : cb) * (kTok * 128);
#pragma unroll
        for (int c = 0; c < 8; ++c) nxt[c] = lds128(nrow + ((c ^ sw) << 4));
        if (FAST) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint32_t w[4] = {cur[c].x, cur[c].y, cur[c].z, cur[c].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float x0 = __uint_as_float(w[q] << 16), x1 = __uint_as_float(w[q] & 0xFFFF0000u);
              pa[c] += x0 + x1;
              pb[c] = fmaf(x0, x0, fmaf(x1, x1, pb[c]));
            }
          }
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c) fold8(cur[c], a, b);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) cur[c] = nxt[c];
      }
      if (FAST) {
        a = ((pa[0] + pa[1]) + (pa[2] + pa[3])) + ((pa[4] + pa[5]) + (pa[6] + pa[7]));
        b = ((pb[0] + pb[1]) + (pb[2] + pb[3])) + ((pb[4] + pb[5]) + (pb[6] + pb[7]));
      }
      if (live) {
        float scale, shift;
        double mu, var;
        row_glue(a, b, m_b * 64, eps, scale, shift, mu, var);
        st[s * kTok + t] = make_float2(scale, shift);
        const int64_t tok = (int64_t)((int)blockIdx.x + i * (int)gridDim.x) * kTok + t;
        if (mean_out) mean_out[tok] = (float)mu;
        if (var_out) var_out[tok] = (float)var;
      }
      __syncwarp();
      if (lane == 0) { if (dbg && blockIdx.x == 0 && (2 * P) < 16) dbg[8 + 5 * (2 * P) + 2] = globaltimer_ns(); }
      if (lane == 0) mbar_arrive(&stat[(2 * P) % stages]);
      if (lane == 16 && 2 * P + 1 < my) mbar_arrive(&stat[(2 * P + 1) % stages]);
    }
  } else {
    // team = kTeamWarps warps = kApplySlabs slabs of 128 chunks: a thread keeps
    // one (token, chunk) position and walks the slabs tid/128 + k*kApplySlabs;
    // team j takes groups j, j + kApplyTeams, ... so per-group waits overlap
    const int aw = warp - 1 - kFoldWarps;
    const int team = aw / kTeamWarps;
    const int tid = (aw % kTeamWarps) * 32 + lane;
    if (m_b * 8 <= kTeamWarps * 32) {
      // feature-stationary mapping (F <= 1024): a thread owns one 8-feature
      // chunk (slab cb, chunk c) for the whole kernel, so its gamma / beta are
      // loaded once into registers, and walks the group's 16 tokens; a warp's
      // 16-byte reads cover 4 full 128-byte rows (conflict-free)
      const int c = tid & 7, cb = tid >> 3;
      const bool own = cb < m_b;
      float g[8], bb[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) { g[e] = 1.0f; bb[e] = 0.0f; }
      if (own) {
        const int f0 = cb * 64 + c * 8;
        if (gamma) {
          const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + f0));
          const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma + f0 + 4));
          g[0] = g0.x; g[1] = g0.y; g[2] = g0.z; g[3] = g0.w; g[4] = g1.x; g[5] = g1.y; g[6] = g1.z; g[7] = g1.w;
        }
        if (beta) {
          const float4 b0 = __ldg(reinterpret_cast<const float4*>(beta + f0));
          const float4 b1 = __ldg(reinterpret_cast<const float4*>(beta + f0 + 4));
          bb[0] = b0.x; bb[1] = b0.y; bb[2] = b0.z; bb[3] = b0.w; bb[4] = b1.x; bb[5] = b1.y; bb[6] = b1.z; bb[7] = b1.w;
        }
      }
      for (int i = team; i < my; i += kApplyTeams) {
        const int s = i % stages;
        LN_WAIT(&full[s], (i / stages) & 1);  // (already complete: the fold waited on it)
        LN_WAIT(&stat[s], (i / stages) & 1);
        if (own) {
          const uint32_t slab = sbase + s * gbytes + cb * (kTok * 128);
#pragma unroll 1
          for (int t0 = 0; t0 < kTok; t0 += 4) {
            uint4 vv[4];
            float2 sc[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int t = t0 + u;
              vv[u] = lds128(slab + t * 128 + ((c ^ (t & 7)) << 4));
              sc[u] = st[s * kTok + t];
            }
            float r[32];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const uint32_t w[4] = {vv[u].x, vv[u].y, vv[u].z, vv[u].w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float x0 = __uint_as_float(w[q] << 16), x1 = __uint_as_float(w[q] & 0xFFFF0000u);
                if (FAST) {
                  const float2 tt = __ffma2_rn(make_float2(x0, x1), make_float2(sc[u].x, sc[u].x),
                                               make_float2(sc[u].y, sc[u].y));
                  const float2 y = __ffma2_rn(tt, make_float2(g[2 * q], g[2 * q + 1]),
                                              make_float2(bb[2 * q], bb[2 * q + 1]));
                  r[8 * u + 2 * q] = y.x;
                  r[8 * u + 2 * q + 1] = y.y;
                } else {
                  // B + (shift + x*scale)*G, every product and sum rounded separately
                  r[8 * u + 2 * q] = __fadd_rn(bb[2 * q], __fmul_rn(__fadd_rn(sc[u].y, __fmul_rn(x0, sc[u].x)), g[2 * q]));
                  r[8 * u + 2 * q + 1] =
                      __fadd_rn(bb[2 * q + 1], __fmul_rn(__fadd_rn(sc[u].y, __fmul_rn(x1, sc[u].x)), g[2 * q + 1]));
                }
              }
            }
            uint32_t o[16];
            pack_bf16_ref_n<16>(r, o);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int t = t0 + u;
              sts128(slab + t * 128 + ((c ^ (t & 7)) << 4), make_uint4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]));
            }
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[s]);
        if (lane == 0 && aw % kTeamWarps == 0) { if (dbg && blockIdx.x == 0 && (i) < 16) dbg[8 + 5 * (i) + 3] = globaltimer_ns(); }
      }
      return;
    }
    const int t = (tid >> 3) & (kTok - 1), c = (tid & 7) ^ (t & 7);
    for (int i = team; i < my; i += kApplyTeams) {
      const int s = i % stages;
      LN_WAIT(&full[s], (i / stages) & 1);  // (already complete: the fold waited on it)
      LN_WAIT(&stat[s], (i / stages) & 1);
      const float2 sc = st[s * kTok + t];
      uint32_t addr = sbase + s * gbytes + tid * 16;
      // 4 chunks per step (slabs cb, cb+2, cb+4, cb+6): their shared-memory
      // loads are in flight together
      for (int cb0 = tid >> 7; cb0 < m_b; cb0 += 4 * kApplySlabs, addr += 4 * kApplySlabs * kTok * 128) {
       uint4 vv[4];
#pragma unroll
       for (int u = 0; u < 4; ++u)
         vv[u] = cb0 + kApplySlabs * u < m_b ? lds128(addr + u * kApplySlabs * kTok * 128) : make_uint4(0, 0, 0, 0);
       float r[32];
#pragma unroll
       for (int u = 0; u < 4; ++u) {
        const int f0 = (cb0 + kApplySlabs * u) * 64 + c * 8;
        float4 g4[2], b4[2];
        if (gamma && cb0 + kApplySlabs * u < m_b) {
          g4[0] = __ldg(reinterpret_cast<const float4*>(gamma + f0));
          g4[1] = __ldg(reinterpret_cast<const float4*>(gamma + f0 + 4));
        } else {
          g4[0] = g4[1] = make_float4(1.0f, 1.0f, 1.0f, 1.0f);
        }
        if (beta && cb0 + kApplySlabs * u < m_b) {
          b4[0] = __ldg(reinterpret_cast<const float4*>(beta + f0));
          b4[1] = __ldg(reinterpret_cast<const float4*>(beta + f0 + 4));
        } else {
          b4[0] = b4[1] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
        const uint32_t w[4] = {vv[u].x, vv[u].y, vv[u].z, vv[u].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          // B + (shift + x*scale)*G, every product and sum rounded separately
          // (scalar: ptxas contracts paired f32x2 mul/add into FFMA2)
          const float x0 = __uint_as_float(w[q] << 16), x1 = __uint_as_float(w[q] & 0xFFFF0000u);
          const float g0 = (q & 1) ? g4[q >> 1].z : g4[q >> 1].x, g1 = (q & 1) ? g4[q >> 1].w : g4[q >> 1].y;
          const float b0 = (q & 1) ? b4[q >> 1].z : b4[q >> 1].x, b1 = (q & 1) ? b4[q >> 1].w : b4[q >> 1].y;
          if (FAST) {
            const float2 t = __ffma2_rn(make_float2(x0, x1), make_float2(sc.x, sc.x), make_float2(sc.y, sc.y));
            const float2 y = __ffma2_rn(t, make_float2(g0, g1), make_float2(b0, b1));
            r[8 * u + 2 * q] = y.x;
            r[8 * u + 2 * q + 1] = y.y;
          } else {
            r[8 * u + 2 * q] = __fadd_rn(b0, __fmul_rn(__fadd_rn(sc.y, __fmul_rn(x0, sc.x)), g0));
            r[8 * u + 2 * q + 1] = __fadd_rn(b1, __fmul_rn(__fadd_rn(sc.y, __fmul_rn(x1, sc.x)), g1));
          }
        }
       }
       // one NaN check for the 32 results, then the 4 stores
       uint32_t o[16];
       pack_bf16_ref_n<16>(r, o);
#pragma unroll
       for (int u = 0; u < 4; ++u)
         if (cb0 + kApplySlabs * u < m_b)
           sts128(addr + u * kApplySlabs * kTok * 128, make_uint4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]));
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&done[s]);
      if (lane == 0 && aw % kTeamWarps == 0) { if (dbg && blockIdx.x == 0 && (i) < 16) dbg[8 + 5 * (i) + 3] = globaltimer_ns(); }
    }
  }
}

static bool ln_simple() {  // experiments: skip the TMA-ring kernel
  static const bool v = getenv("TPP_LN_SIMPLE") != nullptr;
  return v;
}

int launch_layernorm_blocked(int n_b, int m_b, int bn, int bm, int dtype, const void* x,
                             const float* gamma, const float* beta, double eps, void* out,
                             float* mean_out, float* var_out, cudaStream_t s, int exact) {
  const bool al16 = reinterpret_cast<uintptr_t>(x) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(gamma) % 16 == 0 && reinterpret_cast<uintptr_t>(beta) % 16 == 0;
  const int gbytes = lnt::kTok * m_b * 128;
  if (dtype == TPP_BF16 && bm == 64 && bn % lnt::kTok == 0 && al16 && m_b <= 256 &&
      2 * gbytes <= lnt::kRingBytes && !ln_simple()) {
    const int n_groups = n_b * bn / lnt::kTok;
    if (n_groups == 0) return TPP_OK;
    int stages = lnt::kRingBytes / gbytes;
    if (stages > lnt::kMaxStages) stages = lnt::kMaxStages;
    CUtensorMap mx, mo;
    const uint64_t dims[5] = {64, (uint64_t)bn, (uint64_t)m_b, (uint64_t)n_b, 1};
    const uint64_t str[4] = {128, (uint64_t)bn * 128, (uint64_t)m_b * bn * 128, (uint64_t)n_b * m_b * bn * 128};
    const uint32_t box[5] = {64, (uint32_t)lnt::kTok, (uint32_t)m_b, 1, 1};
    int rc = make_tma_map_5d(&mx, x, dims, str, box, 128);
    if (rc) return rc;
    rc = make_tma_map_5d(&mo, out, dims, str, box, 128);
    if (rc) return rc;
    const size_t smem = (size_t)stages * gbytes + 3 * lnt::kMaxStages * 8 + lnt::kMaxStages * lnt::kTok * 8 +
                        lnt::kMaxStages * 4 + 1024;
    {
      cudaError_t e = ensure_smem_attr((const void*)layernorm_blocked_tma<0>, (int)(lnt::kRingBytes + 3 * 1024));
      if (e == cudaSuccess) e = ensure_smem_attr((const void*)layernorm_blocked_tma<1>, (int)(lnt::kRingBytes + 3 * 1024));
      if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(layernorm_blocked_tma)");
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n_groups < num_sms() ? n_groups : num_sms());
    cfg.blockDim = dim3(lnt::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_allowed();
    cfg.attrs = at;
    cfg.numAttrs = 1;
    static const int ln_spin = getenv("TPP_LN_SPIN") ? atoi(getenv("TPP_LN_SPIN")) : 0;  // diagnostics
    cudaError_t e = cudaLaunchKernelEx(&cfg, exact ? layernorm_blocked_tma<0> : layernorm_blocked_tma<1>, mx, mo, n_groups, bn, m_b, stages, gamma, beta,
                                       eps, mean_out, var_out, ln_spin,
                                       debug_timestamps());
    if (e != cudaSuccess) return cuda_status(e, "cudaLaunchKernelEx(layernorm_blocked_tma)");
    TPP_CUDA_LAUNCH_CHECK("layernorm_blocked_tma");
    return TPP_OK;
  }
  if (dtype == TPP_BF16 && bm == 64 && bn % 32 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(out) % 16 == 0 && reinterpret_cast<uintptr_t>(gamma) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(beta) % 16 == 0) {
    const size_t smem = (size_t)32 * (m_b * 8 + 1) * 16 + 64 * sizeof(float);
    if (smem <= 227 * 1024) {
      const int blocks = n_b * (bn / 32);
      if (blocks == 0) return TPP_OK;
      cudaError_t e = ensure_smem_attr((const void*)layernorm_blocked_bf16_v, 227 * 1024);
      if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(layernorm_blocked_bf16_v)");
      layernorm_blocked_bf16_v<<<blocks, 256, smem, s>>>(n_b, m_b, bn, (const uint4*)x, (const float4*)gamma,
                                                         (const float4*)beta, eps,
                                                         (uint4*)out, mean_out, var_out);
      TPP_CUDA_LAUNCH_CHECK("layernorm_blocked_bf16_v");
      return TPP_OK;
    }
  }
  const int F = m_b * bm;
  const int es = dtype == TPP_BF16 ? 2 : 4;
  const int pitch = F + (es == 2 ? 2 : 1);
  const size_t smem = (((size_t)32 * pitch * es + 15) & ~(size_t)15) + 64 * sizeof(float);
  TPP_REQUIRE(smem <= 227 * 1024, TPP_E_UNSUPPORTED, "layernorm_blocked: feature row too long for smem");
  const int blocks = n_b * ((bn + 31) / 32);
  if (blocks == 0) return TPP_OK;
  cudaError_t e;
  if (es == 2) {
    e = ensure_smem_attr((const void*)layernorm_blocked_kernel<uint16_t>, 227 * 1024);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(layernorm_blocked)");
    layernorm_blocked_kernel<uint16_t><<<blocks, 256, smem, s>>>(
        n_b, m_b, bn, bm, (const uint16_t*)x, gamma, beta, eps, (uint16_t*)out, mean_out, var_out);
  } else {
    e = ensure_smem_attr((const void*)layernorm_blocked_kernel<float>, 227 * 1024);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(layernorm_blocked)");
    layernorm_blocked_kernel<float><<<blocks, 256, smem, s>>>(
        n_b, m_b, bn, bm, (const float*)x, gamma, beta, eps, (float*)out, mean_out, var_out);
  }
  TPP_CUDA_LAUNCH_CHECK("layernorm_blocked_kernel");
  return TPP_OK;
}

// ---- softmax (kernels.py:84-99), one CTA per s1 x s3 slice -------------------
__global__ void softmax_kernel(int s1, int s3, DView x, float* y, int y_ld) {
  extern __shared__ float ssm[];  // per-column sums [s3], then reduction scratch
  const int j0 = blockIdx.x * s3;
  // max over the slice (order irrelevant for max; NaN propagates)
  float mx = -__int_as_float(0x7F800000);
  bool nan = false;
  for (int e = threadIdx.x; e < s1 * s3; e += blockDim.x) {
    const float v = nload(x, e % s1, j0 + e / s1);
    if (v != v) nan = true;
    mx = fmaxf(mx, v);
  }
  float* red = ssm + s3;
  red[threadIdx.x] = nan ? __int_as_float(0x7FC00000) : mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = red[0];
    for (int t = 1; t < blockDim.x; ++t) m = (m != m || red[t] != red[t]) ? __int_as_float(0x7FC00000) : fmaxf(m, red[t]);
    red[0] = m;
  }
  __syncthreads();
  mx = red[0];
  // per-column fold over rows ascending (ops.py:519 "per_col")
  for (int c = threadIdx.x; c < s3; c += blockDim.x) {
    float acc = 0.0f;
    for (int i = 0; i < s1; ++i) acc = __fadd_rn(acc, exp_taylor(__fsub_rn(nload(x, i, j0 + c), mx)));
    ssm[c] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.0f;
    for (int c = 0; c < s3; ++c) tot = __fadd_rn(tot, ssm[c]);
    red[1] = __fdiv_rn(1.0f, tot);
  }
  __syncthreads();
  const float rcp = red[1];
  for (int e = threadIdx.x; e < s1 * s3; e += blockDim.x) {
    const int i = e % s1, c = e / s1;
    const float ev = exp_taylor(__fsub_rn(nload(x, i, j0 + c), mx));
    y[i + (int64_t)(j0 + c) * y_ld] = __fmul_rn(ev, rcp);
  }
}

int launch_softmax(int s1, int s2, int s3, const DView& x, float* y, int y_ld, cudaStream_t s) {
  if (s2 == 0) return TPP_OK;
  const int threads = 128;
  const size_t smem = (size_t)(s3 + threads + 2) * sizeof(float);
  TPP_REQUIRE(smem <= 48 * 1024, TPP_E_UNSUPPORTED, "softmax slice too wide");
  softmax_kernel<<<s2, threads, smem, s>>>(s1, s3, x, y, y_ld);
  TPP_CUDA_LAUNCH_CHECK("softmax_kernel");
  return TPP_OK;
}

// ---- split-SGD (kernels.py:235-251): pack, W - g*lr, unpack (bitwise FP32 SGD)
__global__ void split_sgd_kernel(int64_t n, uint16_t* hi, uint16_t* lo, const void* grad,
                                 int grad_dtype, float lr) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float w = __uint_as_float(((uint32_t)hi[e] << 16) | lo[e]);
    const float g = grad_dtype == TPP_BF16 ? bf16_to_f32(reinterpret_cast<const uint16_t*>(grad)[e])
                                           : reinterpret_cast<const float*>(grad)[e];
    const float r = __fsub_rn(w, __fmul_rn(g, lr));
    const uint32_t u = __float_as_uint(r);
    hi[e] = (uint16_t)(u >> 16);
    lo[e] = (uint16_t)(u & 0xFFFF);
  }
}

// 8 parameters per thread-step with 16-byte accesses (FP32 gradients)
__global__ void __launch_bounds__(256)
split_sgd_vec_kernel(int64_t n8, uint4* __restrict__ hi, uint4* __restrict__ lo, const float4* __restrict__ grad,
                     float lr) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n8; e += (int64_t)gridDim.x * blockDim.x) {
    const uint4 h = hi[e], l = lo[e];
    const float4 g0 = __ldg(grad + 2 * e), g1 = __ldg(grad + 2 * e + 1);
    const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[4] = {l.x, l.y, l.z, l.w};
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    uint32_t oh[4], ol[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float w0 = __uint_as_float((hw[q] << 16) | (lw[q] & 0xFFFFu));
      const float w1 = __uint_as_float((hw[q] & 0xFFFF0000u) | (lw[q] >> 16));
      const uint32_t r0 = __float_as_uint(__fsub_rn(w0, __fmul_rn(g[2 * q], lr)));
      const uint32_t r1 = __float_as_uint(__fsub_rn(w1, __fmul_rn(g[2 * q + 1], lr)));
      oh[q] = (r0 >> 16) | (r1 & 0xFFFF0000u);
      ol[q] = (r0 & 0xFFFFu) | (r1 << 16);
    }
    hi[e] = make_uint4(oh[0], oh[1], oh[2], oh[3]);
    lo[e] = make_uint4(ol[0], ol[1], ol[2], ol[3]);
  }
}

// 8 parameters per thread-step with 16-byte accesses (BF16 gradients: the
// exchanged buckets of data-parallel training)
__global__ void __launch_bounds__(256)
split_sgd_vec_bf16_kernel(int64_t n8, uint4* __restrict__ hi, uint4* __restrict__ lo, const uint4* __restrict__ grad,
                          float lr) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n8; e += (int64_t)gridDim.x * blockDim.x) {
    const uint4 h = hi[e], l = lo[e], gv = __ldg(grad + e);
    const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[4] = {l.x, l.y, l.z, l.w}, gw[4] = {gv.x, gv.y, gv.z, gv.w};
    uint32_t oh[4], ol[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float w0 = __uint_as_float((hw[q] << 16) | (lw[q] & 0xFFFFu));
      const float w1 = __uint_as_float((hw[q] & 0xFFFF0000u) | (lw[q] >> 16));
      const float g0 = __uint_as_float(gw[q] << 16), g1 = __uint_as_float(gw[q] & 0xFFFF0000u);
      const uint32_t r0 = __float_as_uint(__fsub_rn(w0, __fmul_rn(g0, lr)));
      const uint32_t r1 = __float_as_uint(__fsub_rn(w1, __fmul_rn(g1, lr)));
      oh[q] = (r0 >> 16) | (r1 & 0xFFFF0000u);
      ol[q] = (r0 & 0xFFFFu) | (r1 << 16);
    }
    hi[e] = make_uint4(oh[0], oh[1], oh[2], oh[3]);
    lo[e] = make_uint4(ol[0], ol[1], ol[2], ol[3]);
  }
}

int launch_split_sgd(int64_t n, uint16_t* hi, uint16_t* lo, const void* grad, int grad_dtype,
                     float lr, cudaStream_t s) {
  if (n == 0) return TPP_OK;
  if (grad_dtype == TPP_BF16 && n % 8 == 0 && reinterpret_cast<uintptr_t>(hi) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(lo) % 16 == 0 && reinterpret_cast<uintptr_t>(grad) % 16 == 0) {
    const int64_t n8 = n / 8;
    int64_t blocks = (n8 + 255) / 256;
    if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
    split_sgd_vec_bf16_kernel<<<(unsigned)blocks, 256, 0, s>>>(n8, reinterpret_cast<uint4*>(hi),
                                                               reinterpret_cast<uint4*>(lo),
                                                               reinterpret_cast<const uint4*>(grad), lr);
    TPP_CUDA_LAUNCH_CHECK("split_sgd_vec_bf16_kernel");
    return TPP_OK;
  }
  if (grad_dtype == TPP_FP32 && n % 8 == 0 && reinterpret_cast<uintptr_t>(hi) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(lo) % 16 == 0 && reinterpret_cast<uintptr_t>(grad) % 16 == 0) {
    const int64_t n8 = n / 8;
    int64_t blocks = (n8 + 255) / 256;
    if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
    split_sgd_vec_kernel<<<(unsigned)blocks, 256, 0, s>>>(n8, reinterpret_cast<uint4*>(hi), reinterpret_cast<uint4*>(lo),
                                                          reinterpret_cast<const float4*>(grad), lr);
    TPP_CUDA_LAUNCH_CHECK("split_sgd_vec_kernel");
    return TPP_OK;
  }
  const int threads = 256;
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > 148 * 32) blocks = 148 * 32;
  split_sgd_kernel<<<(unsigned)blocks, threads, 0, s>>>(n, hi, lo, grad, grad_dtype, lr);
  TPP_CUDA_LAUNCH_CHECK("split_sgd_kernel");
  return TPP_OK;
}

}  // namespace tpp

namespace tpp {

// ---- softmax cross-entropy gradient on blocked logits ------------------------
// Per token: the reference softmax of a 1 x F slice (kernels.py:60-99:
// max-shift, exp_taylor, ascending sum, reciprocal, multiply), then
// dlogit = (p - onehot) * scale and loss = -log(p[target]).
// A CTA stages 16 tokens' logits in smem; the max (order-free), the F
// exponentials and the outputs are computed by all 256 threads; only the
// reference's ascending sum is a per-token serial chain (16 lanes).
constexpr int kXentTok = 16;

__global__ void __launch_bounds__(256)
softmax_xent_blocked_kernel(int n_b, int m_b, int bn, int bm, const float* __restrict__ logits,
                            const int32_t* __restrict__ targets, float scale,
                            uint16_t* __restrict__ dlog, float* __restrict__ loss) {
  extern __shared__ __align__(16) uint8_t xsm[];
  const int F = m_b * bm;
  // row pitch F + 4 floats: 16-byte aligned rows (the serial sum reads
  // float4s), 4-bank skew between consecutive tokens
  const int pitch = F + 4;
  float* rows = reinterpret_cast<float*>(xsm);
  float* mxs = rows + kXentTok * pitch;
  float* rcp = mxs + kXentTok;
  const int chunks_per_blk = (bn + kXentTok - 1) / kXentTok;
  const int nb = blockIdx.x / chunks_per_blk;
  const int n0 = (blockIdx.x % chunks_per_blk) * kXentTok;
  const int T_ = min(kXentTok, bn - n0);
  const int tid = threadIdx.x;
  if (bm == 64 && T_ == kXentTok && blockDim.x == 256) {
    // the cfg-5 shape: each feature block's 16 x 64 sub-tile is 256 float4,
    // one per thread (token t = tid / 16, float4 m4 = tid % 16): no index
    // arithmetic per element, all 16 blocks' loads in flight at once
    const int t = tid >> 4, m4 = tid & 15;
    const float4* src = reinterpret_cast<const float4*>(logits + ((int64_t)nb * m_b * bn + n0) * 64) + tid;
    float* d = rows + t * pitch + m4 * 4;
    for (int mb0 = 0; mb0 < m_b; mb0 += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (mb0 + u < m_b) v[u] = __ldg(src + (int64_t)(mb0 + u) * bn * 16);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (mb0 + u < m_b) {
          float* q = d + (mb0 + u) * 64;
          q[0] = v[u].x; q[1] = v[u].y; q[2] = v[u].z; q[3] = v[u].w;
        }
    }
  } else if (bm % 4 == 0 && (T_ * bm) % 4 == 0) {
    // 16-byte loads, 8 in flight per thread (the logits are read once from HBM)
    const int n4 = T_ * bm / 4, bm4 = bm / 4;
    for (int base = 0; base < m_b * n4; base += 8 * blockDim.x) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = base + u * blockDim.x + tid;
        if (e < m_b * n4) {
          const int mb = e / n4, r4 = e - mb * n4;
          v[u] = __ldg(reinterpret_cast<const float4*>(logits + (((int64_t)nb * m_b + mb) * bn + n0) * bm) + r4);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = base + u * blockDim.x + tid;
        if (e < m_b * n4) {
          const int mb = e / n4, r4 = e - mb * n4, t = r4 / bm4, m = (r4 - t * bm4) * 4;
          float* d = rows + t * pitch + mb * bm + m;
          d[0] = v[u].x; d[1] = v[u].y; d[2] = v[u].z; d[3] = v[u].w;
        }
      }
    }
  } else {
    for (int mb = 0; mb < m_b; ++mb) {
      const float* src = logits + (((int64_t)nb * m_b + mb) * bn + n0) * bm;
      for (int e = tid; e < T_ * bm; e += blockDim.x) {
        const int t = e / bm, m = e - t * bm;
        rows[t * pitch + mb * bm + m] = __ldg(src + e);
      }
    }
  }
  __syncthreads();
  // max over the slice (np.max: NaN if any element is NaN): 16 threads per token
  {
    const int t = tid >> 4, k = tid & 15;
    float mx = -__int_as_float(0x7F800000);
    bool nan = false;
    if (t < T_) {
      const float* r = rows + t * pitch;
      for (int f = k; f < F; f += 16) {
        const float v = r[f];
        nan |= v != v;
        mx = fmaxf(mx, v);
      }
    }
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
      mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
      nan |= __shfl_xor_sync(0xFFFFFFFFu, (int)nan, o) != 0;
    }
    if (k == 0 && t < T_) mxs[t] = nan ? __int_as_float(0x7FC00000) : mx;
  }
  __syncthreads();
  // e = exp_taylor(x - max), in place: 16 threads per token, no index division
  {
    const int t = tid >> 4, k = tid & 15;
    if (t < T_) {
      float* r = rows + t * pitch;
      const float mx = mxs[t];
#pragma unroll 4
      for (int f = k; f < F; f += 16) r[f] = exp_taylor(__fsub_rn(r[f], mx));
    }
  }
  __syncthreads();
  // the reference's ascending sum: one serial chain per token
  if (tid < T_) {
    const float* r = rows + tid * pitch;
    float tot = 0.0f;
    int f = 0;
    if (F % 16 == 0 && F >= 16) {
      // float4 reads one 16-float chunk ahead of the dependent add chain
      const float4* r4 = reinterpret_cast<const float4*>(r);
      float4 a0 = r4[0], a1 = r4[1], a2 = r4[2], a3 = r4[3];
      for (; f < F; f += 16) {
        float4 n0 = a0, n1 = a1, n2 = a2, n3 = a3;
        if (f + 16 < F) {
          const float4* q = r4 + (f + 16) / 4;
          n0 = q[0]; n1 = q[1]; n2 = q[2]; n3 = q[3];
        }
        const float v[16] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w,
                             a2.x, a2.y, a2.z, a2.w, a3.x, a3.y, a3.z, a3.w};
#pragma unroll
        for (int u = 0; u < 16; ++u) tot = __fadd_rn(tot, v[u]);
        a0 = n0; a1 = n1; a2 = n2; a3 = n3;
      }
    }
    for (; f + 8 <= F; f += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = r[f + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) tot = __fadd_rn(tot, v[u]);
    }
    for (; f < F; ++f) tot = __fadd_rn(tot, r[f]);
    const float rc = __fdiv_rn(1.0f, tot);
    rcp[tid] = rc;
    const int64_t tok = (int64_t)nb * bn + n0 + tid;
    if (loss) loss[tok] = -logf(__fmul_rn(r[targets[tok]], rc));
  }
  __syncthreads();
  // dlogits: 16 threads per token, 4 consecutive features each (8-byte stores)
  if (bm == 64 && T_ == kXentTok && blockDim.x == 256) {
    // same mapping as the load: per feature block one 8-byte store per thread,
    // a warp writes two token rows of 128 contiguous bytes
    const int t = tid >> 4, m4 = tid & 15;
    const float rc = rcp[t];
    const int tg = targets[(int64_t)nb * bn + n0 + t];
    const float* r = rows + t * pitch + m4 * 4;
    uint2* dst = reinterpret_cast<uint2*>(dlog + ((int64_t)nb * m_b * bn + n0) * 64) + tid;
#pragma unroll 4
    for (int mb = 0; mb < m_b; ++mb) {
      const int f = mb * 64 + m4 * 4;
      float g[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        g[u] = __fmul_rn(__fsub_rn(__fmul_rn(r[mb * 64 + u], rc), f + u == tg ? 1.0f : 0.0f), scale);
      uint32_t w[2];
      pack_bf16_ref_n<2>(g, w);   // hardware RNE, one rarely-taken branch for the NaN rule
      dst[(int64_t)mb * bn * 16] = make_uint2(w[0], w[1]);
    }
  } else if (bm % 64 == 0) {
    const int t = tid >> 4, k = tid & 15;
    if (t < T_) {
      const float rc = rcp[t];
      const int tg = targets[(int64_t)nb * bn + n0 + t];
      const float* r = rows + t * pitch;
      for (int mb = 0; mb < m_b; ++mb) {
        uint16_t* dst = dlog + ((((int64_t)nb * m_b + mb) * bn + n0 + t) * bm);
        for (int m = 4 * k; m < bm; m += 64) {
          const int f = mb * bm + m;
          float g[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            g[u] = __fmul_rn(__fsub_rn(__fmul_rn(r[f + u], rc), f + u == tg ? 1.0f : 0.0f), scale);
          *reinterpret_cast<uint2*>(dst + m) = make_uint2(pack2_bf16_ref(g[0], g[1]), pack2_bf16_ref(g[2], g[3]));
        }
      }
    }
  } else {
    for (int mb = 0; mb < m_b; ++mb) {
      uint16_t* dst = dlog + (((int64_t)nb * m_b + mb) * bn + n0) * bm;
      for (int e = tid; e < T_ * bm; e += blockDim.x) {
        const int t = e / bm, m = e - t * bm;
        const int f = mb * bm + m;
        const float pr = __fmul_rn(rows[t * pitch + f], rcp[t]);
        const int tg = targets[(int64_t)nb * bn + n0 + t];
        const float g = __fmul_rn(__fsub_rn(pr, f == tg ? 1.0f : 0.0f), scale);
        dst[e] = f32_to_bf16(g);
      }
    }
  }
}

// ---- softmax-CE with every token of an SM resident -------------------------
// The reference's per-token sum is a 1024-long dependent FADD chain (~4k
// cycles).  In the 16-token kernel above every other warp of the CTA waits at
// a barrier while 16 lanes run it (ncu: 28 % of the warp samples on that
// barrier, 1.15 waves of 3 CTAs per SM, DRAM 13 % busy).  Here one CTA per SM
// owns <= 56 consecutive tokens, all resident in smem at once (56 x 4 KB):
//   warps 2-15  copy every token's logits into smem at once (cp.async, each
//               thread the 16-byte quads it reads later: the whole SM share
//               in flight); per token (a half warp, 16 float4 per lane in
//               registers): max (16-lane shuffle), exp_taylor, exponentials
//               back to smem -- tokens 0-27 first, so their sums overlap the
//               second round's exponentials; then each round's dlogits once
//               its sums are done
//   warps 0, 1  the serial sums of tokens 0-27 / 28-55 (lane = token).
// (256-byte TMA bulk copies per token row measured slower: 58 vs 38 us.)
// Same arithmetic and order as the kernel above (bitwise).
constexpr int kXpThreads = 512;
constexpr int kXpWorkers = kXpThreads - 64;       // 14 warps = 28 token rows per round
constexpr int kXpRound = kXpWorkers / 16;          // 28
constexpr int kXpMaxTok = 2 * kXpRound;            // 56

__global__ void __launch_bounds__(kXpThreads, 1)
softmax_xent_resident_kernel(int n_tok, int m_b, int bn, const float* __restrict__ logits,
                             const int32_t* __restrict__ targets, float scale, uint16_t* __restrict__ dlog,
                             float* __restrict__ loss) {
  using namespace sm100;
  extern __shared__ __align__(16) uint8_t xsm[];
  const int F = m_b * 64;
  const int pitch = F + 4;  // floats; 16-byte aligned rows, 4-bank skew per token
  float* rows = reinterpret_cast<float*>(xsm);
  float* rcs = rows + kXpMaxTok * pitch;
  uint64_t* exp_ready = reinterpret_cast<uint64_t*>(rcs + kXpMaxTok);  // [2] round's exponentials written
  uint64_t* sum_ready = exp_ready + 2;                                // [2] round's sums done
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t_begin = (int)(((int64_t)n_tok * blockIdx.x) / gridDim.x);
  const int ntok = (int)(((int64_t)n_tok * (blockIdx.x + 1)) / gridDim.x) - t_begin;   // <= 56
  const int nr0 = min(ntok, kXpRound), nr1 = ntok - nr0;
  if (threadIdx.x == 0) {
    for (int c = 0; c < 2; ++c) {
      mbar_init(&exp_ready[c], c == 0 ? max(nr0, 1) : max(nr1, 1));  // one arrival per token
      mbar_init(&sum_ready[c], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp <= 1) {
    // ===== the reference's ascending sums: round `warp`, one lane per token =====
    const int c = warp, nrc = c == 0 ? nr0 : nr1;
    if (nrc > 0) {
      mbar_wait_sleep(&exp_ready[c], 0);   // sleeping: the workers need the issue slots
      if (lane < nrc) {
        const int t = c * kXpRound + lane;
        const float* r = rows + t * pitch;
        float tot = 0.0f;
        const float4* r4 = reinterpret_cast<const float4*>(r);
        float4 a0 = r4[0], a1 = r4[1], a2 = r4[2], a3 = r4[3];
        for (int f = 0; f < F; f += 16) {   // F % 64 == 0: float4 reads one 16-float chunk ahead
          float4 n0 = a0, n1 = a1, n2 = a2, n3 = a3;
          if (f + 16 < F) {
            const float4* q = r4 + (f + 16) / 4;
            n0 = q[0]; n1 = q[1]; n2 = q[2]; n3 = q[3];
          }
          const float v[16] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w,
                               a2.x, a2.y, a2.z, a2.w, a3.x, a3.y, a3.z, a3.w};
#pragma unroll
          for (int u = 0; u < 16; ++u) tot = __fadd_rn(tot, v[u]);
          a0 = n0; a1 = n1; a2 = n2; a3 = n3;
        }
        const float rc = __fdiv_rn(1.0f, tot);
        rcs[t] = rc;
        const int tok = t_begin + t;
        if (loss) loss[tok] = -logf(__fmul_rn(r[targets[tok]], rc));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sum_ready[c]);
    }
    return;
  }
  // ===== workers: half warp = one token row, lane m4 = feature quad m4 of every block =====
  const int wt = threadIdx.x - 64;
  const int tr = wt >> 4, m4 = wt & 15;
  // the whole SM share in flight at once: each thread copies (cp.async, 16 B)
  // exactly the quads it later reads -- its token of each round -- so its own
  // wait_group is the only synchronisation a round's loads need
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int t = c * kXpRound + tr;
    if (t < ntok) {
      const int tok = t_begin + t, nb = tok / bn, nin = tok - nb * bn;
      const float* src = logits + ((int64_t)nb * m_b * bn + nin) * 64 + 4 * m4;
      const uint32_t dst = smem_u32(rows + t * pitch + 4 * m4);
      for (int mb = 0; mb < m_b; ++mb)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + mb * 256),
                     "l"(src + (int64_t)mb * bn * 64)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int c = 0; c < 2; ++c) {
    const int t = c * kXpRound + tr;
    const bool valid = t < ntok;
    float4 v[16];
    float mx = -__int_as_float(0x7F800000);
    bool nan = false;
    if (c == 0) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (valid) {
      const float* row = rows + t * pitch + 4 * m4;
#pragma unroll
      for (int mb = 0; mb < 16; ++mb)
        if (mb < m_b) v[mb] = *reinterpret_cast<const float4*>(row + mb * 64);
#pragma unroll
      for (int mb = 0; mb < 16; ++mb)
        if (mb < m_b) {
          nan |= (v[mb].x != v[mb].x) | (v[mb].y != v[mb].y) | (v[mb].z != v[mb].z) | (v[mb].w != v[mb].w);
          mx = fmaxf(fmaxf(mx, v[mb].x), fmaxf(v[mb].y, fmaxf(v[mb].z, v[mb].w)));
        }
    }
    // (a warp holds two token rows: both halves shuffle even when one is past the end)
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) {
      mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
      nan |= __shfl_xor_sync(0xFFFFFFFFu, (int)nan, o) != 0;
    }
    if (nan) mx = __int_as_float(0x7FC00000);
    if (valid) {
      float* row = rows + t * pitch + 4 * m4;
#pragma unroll
      for (int mb = 0; mb < 16; ++mb)
        if (mb < m_b) {
          float4 e;
          e.x = exp_taylor_nonpos(__fsub_rn(v[mb].x, mx));
          e.y = exp_taylor_nonpos(__fsub_rn(v[mb].y, mx));
          e.z = exp_taylor_nonpos(__fsub_rn(v[mb].z, mx));
          e.w = exp_taylor_nonpos(__fsub_rn(v[mb].w, mx));
          *reinterpret_cast<float4*>(row + mb * 64) = e;
        }
    }
    __syncwarp();
    if (valid && m4 == 0) mbar_arrive(&exp_ready[c]);   // one arrival per token (after its 16 lanes' writes)
  }
  // dlogits of each round once its sums are done
  for (int c = 0; c < 2; ++c) {
    const int t = c * kXpRound + tr;
    if ((c == 0 ? nr0 : nr1) == 0) break;
    mbar_wait_sleep(&sum_ready[c], 0);
    if (t < ntok) {
      const int tok = t_begin + t, nb = tok / bn, nin = tok - nb * bn;
      const float rc = rcs[t];
      const int tg = targets[tok];
      const float* row = rows + t * pitch + 4 * m4;
      uint2* dst = reinterpret_cast<uint2*>(dlog) + ((int64_t)nb * m_b * bn + nin) * 16 + m4;
#pragma unroll 4
      for (int mb = 0; mb < m_b; ++mb) {
        const float4 x = *reinterpret_cast<const float4*>(row + mb * 64);
        const int f = mb * 64 + 4 * m4;
        const float xv[4] = {x.x, x.y, x.z, x.w};
        float g[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          g[u] = __fmul_rn(__fsub_rn(__fmul_rn(xv[u], rc), f + u == tg ? 1.0f : 0.0f), scale);
        uint32_t w[2];
        pack_bf16_ref_n<2>(g, w);
        dst[(int64_t)mb * bn * 16] = make_uint2(w[0], w[1]);
      }
    }
  }
}

int launch_softmax_xent_blocked(int n_b, int m_b, int bn, int bm, const float* logits,
                                const int32_t* targets, float scale, void* dlogits, float* loss,
                                cudaStream_t s) {
  const int F = m_b * bm;
  // every token of an SM resident (bm = 64, <= 16 feature blocks, <= 56 tokens per CTA)
  {
    const int64_t n_tok = (int64_t)n_b * bn;
    static const bool legacy = getenv("TPP_XENT_LEGACY") != nullptr;  // A/B: the 16-token kernel
    const int64_t grid = std::max<int64_t>(num_sms(), (n_tok + kXpMaxTok - 1) / kXpMaxTok);
    if (!legacy && bm == 64 && m_b <= 16 && n_tok >= num_sms() && grid < 65536 &&
        reinterpret_cast<uintptr_t>(logits) % 16 == 0 && reinterpret_cast<uintptr_t>(dlogits) % 8 == 0) {
      const size_t smem = (size_t)kXpMaxTok * (F + 4) * sizeof(float) + kXpMaxTok * sizeof(float) +
                          4 * sizeof(uint64_t);
      cudaError_t e = ensure_smem_attr((const void*)softmax_xent_resident_kernel, (int)smem);
      if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(softmax_xent_resident)");
      softmax_xent_resident_kernel<<<(unsigned)grid, kXpThreads, smem, s>>>(
          (int)n_tok, m_b, bn, logits, targets, scale, reinterpret_cast<uint16_t*>(dlogits), loss);
      TPP_CUDA_LAUNCH_CHECK("softmax_xent_resident_kernel");
      return TPP_OK;
    }
  }
  const size_t smem = (size_t)kXentTok * (F + 4) * sizeof(float) + 2 * kXentTok * sizeof(float);
  TPP_REQUIRE(smem <= 227 * 1024, TPP_E_UNSUPPORTED, "softmax_xent: class dimension too long for smem");
  const int blocks = n_b * ((bn + kXentTok - 1) / kXentTok);
  if (blocks == 0) return TPP_OK;
  cudaError_t e = ensure_smem_attr((const void*)softmax_xent_blocked_kernel, 227 * 1024);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(softmax_xent)");
  softmax_xent_blocked_kernel<<<blocks, 256, smem, s>>>(n_b, m_b, bn, bm, logits, targets, scale,
                                                         reinterpret_cast<uint16_t*>(dlogits), loss);
  TPP_CUDA_LAUNCH_CHECK("softmax_xent_blocked_kernel");
  return TPP_OK;
}

}  // namespace tpp

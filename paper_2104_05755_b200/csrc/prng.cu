// K8: PRNG / DROPOUT / DROPOUT_INV TPPs (ops.py:195-236, 326-328, 378-382, 416-444).
//
// The reference keeps one Marsaglia xorshift128 stream per column, seeded as
// splitmix64(seed ^ col) (ops.py:195-221), and draws row i of a call from the
// (i+1)-th step of every stream (uniform_block, ops.py:230-236).  Each stream
// is a serial recurrence over rows, so a one-thread-per-column kernel would
// expose only `cols` threads and walk columns with strided (uncoalesced)
// accesses.  Instead:
//
//   * xorshift128 is linear over GF(2), so "advance n steps" is a fixed
//     128x128 bit matrix.  The host builds M^(64 * 2^b) once (by squaring)
//     and parks the matrices in constant memory.
//   * work item = 32 columns x (8 * run) rows; lane = column, warp w owns the
//     `run` contiguous rows [w * run, (w + 1) * run) of the item.  A thread
//     jumps its column's stream to its first row ONCE (popcount(row / 64)
//     mat-vecs, constant loads broadcast because the warp shares the row)
//     and then steps through its whole run; `run` is sized on the host so
//     there are ~3 items per SM.
//   * the run is consumed 64 rows at a time: every warp draws 64 rows into
//     shared memory (keep bits for DROPOUT, uniforms for PRNG), then the CTA
//     streams that 32 x (8 x 64) slab with consecutive threads on
//     consecutive 8-row groups of a column (16-byte vector loads/stores).
//     Several CTAs per SM drift out of phase, so one CTA's draws overlap
//     another's HBM streaming.
//   * the stream state is SoA [4][cols] (x, y, z, w rows); a call reads
//     state_in and the thread holding a column's last row writes the advanced
//     stream to state_out (a separate buffer: other CTAs still read state_in).
//
// Numerics are the reference's: u = (w >> 8) * 2^-24 in FP32 (exact), keep =
// u >= float32(p) (== (w >> 8) >= ceil(float32(p) * 2^24), exact), scale =
// compute_dtype(1 / (1 - p)) with 1/(1-p) in double, r = keep ? x * scale : +0
// rounded once into the output dtype.

#include "common.cuh"
#include "sm100.cuh"

#include <algorithm>
#include <cmath>
#include <mutex>

namespace tpp {

namespace {

#ifndef TPP_DRAW_UNROLL
#define TPP_DRAW_UNROLL 8
#endif
#ifndef TPP_DROP_NS
#define TPP_DROP_NS 2
#endif
#ifndef TPP_DROP_STAGES
#define TPP_DROP_STAGES 3
#endif
#ifndef TPP_DROP_MINB
#define TPP_DROP_MINB 1
#endif
constexpr int kDrawUnroll = TPP_DRAW_UNROLL;
constexpr int kSub = 64;                    // rows per draw slab (one keep word)
constexpr int kWarps = 8;
constexpr int kTileCols = 32;
constexpr int kLevels = 26;                 // jumps up to 64 * 2^26 rows
constexpr int kFillStride = kSub * kWarps + 1;  // 513: conflict-free column writes

// Jump tables, four bits at a time: nib[b][p][v] = M^(64 * 2^b) applied to the
// state whose only non-zero bits are v at bit positions 4p .. 4p+3 (word p/8).
// A jump is 32 table loads XOR-ed together (L1-resident, 213 KB total).
constexpr int kNibs = 32;

struct Xs128 {
  uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ uint32_t xs_step(Xs128& s) {
  const uint32_t t = s.x ^ (s.x << 11);
  s.x = s.y;
  s.y = s.z;
  s.z = s.w;
  s.w = (s.w ^ (s.w >> 19)) ^ (t ^ (t >> 8));
  return s.w;
}

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ Xs128 jump(const Xs128& s, const uint4* __restrict__ lvl) {
  const uint32_t words[4] = {s.x, s.y, s.z, s.w};
  uint4 e[kNibs];
#pragma unroll
  for (int p = 0; p < kNibs; ++p) e[p] = __ldg(lvl + p * 16 + ((words[p >> 3] >> ((p & 7) * 4)) & 15u));
  uint32_t ax = 0, ay = 0, az = 0, aw = 0;
#pragma unroll
  for (int p = 0; p < kNibs; ++p) {
    ax ^= e[p].x;
    ay ^= e[p].y;
    az ^= e[p].z;
    aw ^= e[p].w;
  }
  return Xs128{ax, ay, az, aw};
}

// ---- host: jump tables ------------------------------------------------------
struct HostTables {
  uint32_t lvl[kLevels][128][4];
};

static void matvec(const uint32_t (*m)[4], const uint32_t v[4], uint32_t out[4]) {
  out[0] = out[1] = out[2] = out[3] = 0;
  for (int k = 0; k < 128; ++k)
    if ((v[k >> 5] >> (k & 31)) & 1u)
      for (int q = 0; q < 4; ++q) out[q] ^= m[k][q];
}

// c = a * b (apply b, then a)
static void matmul(const uint32_t (*a)[4], const uint32_t (*b)[4], uint32_t (*c)[4]) {
  for (int k = 0; k < 128; ++k) matvec(a, b[k], c[k]);
}

static const HostTables& host_tables() {
  static HostTables* ht = [] {
    HostTables* h = new HostTables();
    for (int k = 0; k < 128; ++k) {
      Xs128 s{0, 0, 0, 0};
      (&s.x)[k >> 5] = 1u << (k & 31);
      for (int i = 0; i < kSub; ++i) xs_step(s);
      h->lvl[0][k][0] = s.x;
      h->lvl[0][k][1] = s.y;
      h->lvl[0][k][2] = s.z;
      h->lvl[0][k][3] = s.w;
    }
    for (int b = 1; b < kLevels; ++b) matmul(h->lvl[b - 1], h->lvl[b - 1], h->lvl[b]);
    return h;
  }();
  return *ht;
}

// Per-device copy of the nibble tables; uploaded on first use (PrngState
// creation calls this too, so a later graph capture finds them resident).
static const uint4* jump_tables(int* rc) {
  static std::mutex mu;
  static const uint4* dev_tab[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || dev >= 64) {
    *rc = cuda_status(e == cudaSuccess ? cudaErrorInvalidDevice : e, "cudaGetDevice");
    return nullptr;
  }
  std::lock_guard<std::mutex> g(mu);
  if (dev_tab[dev]) return dev_tab[dev];
  const HostTables& h = host_tables();
  static uint32_t nib[kLevels][kNibs][16][4];
  for (int b = 0; b < kLevels; ++b)
    for (int p = 0; p < kNibs; ++p)
      for (int v = 0; v < 16; ++v) {
        uint32_t acc[4] = {0, 0, 0, 0};
        for (int t = 0; t < 4; ++t)
          if ((v >> t) & 1)
            for (int q = 0; q < 4; ++q) acc[q] ^= h.lvl[b][4 * p + t][q];
        memcpy(nib[b][p][v], acc, sizeof(acc));
      }
  void* d = nullptr;
  e = cudaMalloc(&d, sizeof(nib));
  if (e == cudaSuccess) e = cudaMemcpy(d, nib, sizeof(nib), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (d) cudaFree(d);
    *rc = cuda_status(e, "prng jump tables");
    return nullptr;
  }
  dev_tab[dev] = reinterpret_cast<const uint4*>(d);
  return dev_tab[dev];
}

// ---- device -----------------------------------------------------------------
__global__ void prng_seed_kernel(uint64_t seed, int cols, uint32_t* state) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  const uint64_t a = splitmix64((uint64_t)j ^ seed);
  const uint64_t b = splitmix64(a);
  uint32_t x = (uint32_t)a, y = (uint32_t)(a >> 32), z = (uint32_t)b, w = (uint32_t)(b >> 32);
  if ((x | y | z | w) == 0) w = 1;  // a stream is never all-zero (ops.py:219-221)
  state[j] = x;
  state[cols + j] = y;
  state[2 * cols + j] = z;
  state[3 * cols + j] = w;
}

template <typename T>
__host__ __device__ __forceinline__ T compute_scale(double p) {
  return (T)(1.0 / (1.0 - p));
}

// 8 consecutive rows [i0, i0 + 8) of column j; vec: 16-byte aligned FP32/BF16
// dense data with all 8 rows in range.
template <typename T>
__device__ __forceinline__ void load8(const DView& in, int i0, int j, int rows, bool vec, T (&x)[8]) {
  if (vec) {
    const int64_t idx = i0 + (int64_t)j * in.ld;
    if (in.dtype == TPP_FP32) {
      const float4 a = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(in.p) + idx)[0];
      const float4 b = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(in.p) + idx)[1];
      x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
    } else {
      const uint4 u = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(in.p) + idx);
      const uint32_t wv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        x[2 * e] = __uint_as_float(wv[e] << 16);
        x[2 * e + 1] = __uint_as_float(wv[e] & 0xFFFF0000u);
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) x[e] = (i0 + e < rows) ? load_elem<T>(in, i0 + e, j) : T(0);
  }
}

template <typename T>
__device__ __forceinline__ void store8(void* out, int out_dtype, int out_ld, int i0, int j, int rows, bool vec,
                                       const T (&r)[8]) {
  const int64_t idx = i0 + (int64_t)j * out_ld;
  if (vec) {
    if (out_dtype == TPP_FP32) {
      float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + idx);
      o[0] = make_float4(r[0], r[1], r[2], r[3]);
      o[1] = make_float4(r[4], r[5], r[6], r[7]);
    } else {
      float f[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = (float)r[e];
      uint32_t u[4];
      pack_bf16_ref_n<4>(f, u);  // hardware RNE, reference NaN rule on the rare NaN path
      *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(out) + idx) = make_uint4(u[0], u[1], u[2], u[3]);
    }
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (i0 + e < rows) store_elem<T>(out, out_dtype, idx + e, r[e]);
  }
}

template <typename T>
__device__ __forceinline__ void scale8(uint32_t byte, T scale, T (&x)[8]) {
#pragma unroll
  for (int e = 0; e < 8; ++e) x[e] = ((byte >> e) & 1u) ? mul_rn(x[e], scale) : T(0);
}

// 64 draws -> keep bits (row i -> bit i); full: all 64 rows in range
// Device step with the right shifts as mul.hi (FMA pipe) so the ALU pipe only
// carries the XORs: the mask draw is ALU-bound otherwise.
__device__ __forceinline__ uint32_t mulhi_u32(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t xs_step_fast(Xs128& s) {
  const uint32_t t = s.x ^ (s.x << 11);
  s.x = s.y;
  s.y = s.z;
  s.z = s.w;
  s.w = (s.w ^ mulhi_u32(s.w, 1u << 13)) ^ (t ^ mulhi_u32(t, 1u << 24));  // >> 19, >> 8
  return s.w;
}

// 32 draws -> keep bits, row i -> bit i.  keep <=> w >= thr (thr = thr24 << 8,
// 0 < thr24 < 2^24) <=> carry(w + (2^32 - thr)); lo = 2 lo + carry puts the
// first row in the MSB, so the word is bit-reversed at the end.
__device__ __forceinline__ uint32_t draw_keep32(Xs128& s, uint32_t nthr) {
  uint32_t lo = 0;
#pragma unroll kDrawUnroll
  for (int i = 0; i < 32; ++i) {
    const uint32_t w = xs_step_fast(s);
    asm("{ .reg .u32 d; add.cc.u32 d, %1, %2; addc.u32 %0, %0, %0; }" : "+r"(lo) : "r"(w), "r"(nthr));
  }
  return __brev(lo);
}

// (w >> 8) >= thr24 <=> w >= thr24 * 256 for thr24 < 2^24; thr24 == 2^24 never keeps.
__device__ __forceinline__ uint64_t draw_keep64(Xs128& s, uint32_t thr24, int n) {
  if (thr24 >= (1u << 24) || thr24 == 0) {
    for (int i = 0; i < n; ++i) xs_step_fast(s);
    return thr24 == 0 ? (n == kSub ? ~0ull : ((1ull << n) - 1)) : 0ull;
  }
  if (n == kSub) {
    const uint32_t nthr = 0u - (thr24 << 8);
    const uint32_t lo = draw_keep32(s, nthr);
    const uint32_t hi = draw_keep32(s, nthr);
    return (uint64_t)lo | ((uint64_t)hi << 32);
  }
  const uint32_t thr = thr24 << 8;
  uint32_t lo = 0, hi = 0;
  for (int i = 0; i < n; ++i) {
    const uint32_t b = (uint32_t)(xs_step_fast(s) >= thr);
    if (i < 32) lo |= b << i;
    else hi |= b << (i - 32);
  }
  return (uint64_t)lo | ((uint64_t)hi << 32);
}

__device__ __forceinline__ Xs128 start_state(const uint32_t* st, int cols, int j, int row,
                                             const uint4* __restrict__ tab) {
  Xs128 s{st[j], st[cols + j], st[2 * cols + j], st[3 * cols + j]};
  for (int b = 0, seg = row / kSub; seg != 0; ++b, seg >>= 1)
    if (seg & 1) s = jump(s, tab + b * kNibs * 16);
  return s;
}

// DROPOUT step 1 (ops.py:430-441): keep bitmask only.  Warp = 32 consecutive
// columns x one run of `run` rows (a multiple of 64); one jump, then `run`
// steps, one 8-byte mask store per 64 rows.  Step 2 is DROPOUT_INV on the
// freshly drawn mask (same keep ? x * scale : 0 per element).
__global__ void __launch_bounds__(256) dropout_mask_kernel(const uint32_t* __restrict__ st_in,
                                                           uint32_t* __restrict__ st_out, uint32_t thr24,
                                                           uint8_t* __restrict__ mask_out, int rows, int cols,
                                                           int run, int mask8, const uint4* __restrict__ tab) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j = blockIdx.x * kTileCols + lane;
  const int64_t rs64 = ((int64_t)blockIdx.y * kWarps + w) * run;
  if (j >= cols || rs64 >= rows) return;
  const int rs = (int)rs64;
  const int nr = min(run, rows - rs);
  Xs128 s = start_state(st_in, cols, j, rs, tab);
  const int bpc = (rows + 7) >> 3;
  uint8_t* mb = mask_out + (int64_t)j * bpc + (rs >> 3);
#pragma unroll 1
  for (int q = 0; q * kSub < nr; ++q) {
    const int n = min(kSub, nr - q * kSub);
    const uint64_t bits = draw_keep64(s, thr24, n);
    // mask layout (tensor.py:246-254): column j owns bpc bytes; row i is bit i&7 of byte i>>3
    if (n == kSub && mask8) {
      *reinterpret_cast<uint64_t*>(mb + q * 8) = bits;
    } else {
      for (int b = 0; b < (n + 7) >> 3; ++b) mb[q * 8 + b] = (uint8_t)(bits >> (8 * b));
    }
  }
  if (rs + nr == rows) {  // this thread drew the column's last row
    st_out[j] = s.x;
    st_out[cols + j] = s.y;
    st_out[2 * cols + j] = s.z;
    st_out[3 * cols + j] = s.w;
  }
}

// DROPOUT fused (dense BF16 / FP32 column-major views, rows % 64 == 0): the
// keep draws and the scaled copy in ONE pass.  Lane = column for the draws
// (warp = 32 columns x a run of `run` rows, one jump, as
// dropout_mask_kernel); the data moves coalesced instead: per 64-row slab the
// warp's 32 x 64 block is read as 8 passes of 4 columns x 64 rows (8 lanes
// per column, 16 contiguous bytes each), issued BEFORE the slab's draws so
// the HBM reads are in flight while the ALU runs the xorshift steps (BF16:
// one slab ahead); each lane fetches its columns' keep byte from the drawing
// lane with a shuffle, applies keep ? x * scale : 0 (the DROPOUT_INV rule,
// FP32 math, RNE + the reference NaN rule for BF16) and stores 16 bytes; the
// drawing lane stores its 8-byte mask word.  Bitwise the mask kernel +
// DROPOUT_INV.
template <typename TI>
struct SlabPart;
template <>
struct SlabPart<uint16_t> {  // 8 rows of BF16 = 16 B per lane per pass
  static constexpr int N = 1;
  uint4 v[8];
  __device__ __forceinline__ void load(const uint16_t* p, int64_t col_stride, bool ok) {
#pragma unroll
    for (int it = 0; it < 8; ++it)
      v[it] = ok ? __ldg(reinterpret_cast<const uint4*>(p + it * 4 * col_stride)) : make_uint4(0, 0, 0, 0);
  }
  __device__ __forceinline__ void get(int it, float (&x)[8]) const {
    const uint32_t w[4] = {v[it].x, v[it].y, v[it].z, v[it].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      x[2 * q] = __uint_as_float(w[q] << 16);
      x[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
    }
  }
};
template <>
struct SlabPart<float> {  // 8 rows of FP32 = 32 B per lane per pass
  float4 v[16];
  __device__ __forceinline__ void load(const float* p, int64_t col_stride, bool ok) {
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const float4* q = reinterpret_cast<const float4*>(p + it * 4 * col_stride);
      v[2 * it] = ok ? __ldg(q) : make_float4(0, 0, 0, 0);
      v[2 * it + 1] = ok ? __ldg(q + 1) : make_float4(0, 0, 0, 0);
    }
  }
  __device__ __forceinline__ void get(int it, float (&x)[8]) const {
    const float4 a = v[2 * it], b = v[2 * it + 1];
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  }
};

template <typename TO>
__device__ __forceinline__ void store8_vec(TO* op, const float (&r)[8]) {
  if constexpr (sizeof(TO) == 2) {
    uint32_t u[4];
    pack_bf16_ref_n<4>(r, u);
    *reinterpret_cast<uint4*>(op) = make_uint4(u[0], u[1], u[2], u[3]);
  } else {
    reinterpret_cast<float4*>(op)[0] = make_float4(r[0], r[1], r[2], r[3]);
    reinterpret_cast<float4*>(op)[1] = make_float4(r[4], r[5], r[6], r[7]);
  }
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(256, TPP_DROP_MINB) dropout_fused_kernel(const uint32_t* __restrict__ st_in,
                                                            uint32_t* __restrict__ st_out, uint32_t thr24,
                                                            const TI* __restrict__ in, TO* __restrict__ out,
                                                            uint8_t* __restrict__ mask_out, int rows, int cols,
                                                            int run, float scale, const uint4* __restrict__ tab) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j0 = blockIdx.x * kTileCols;
  const int j = j0 + lane;
  const int64_t rs64 = ((int64_t)blockIdx.y * kWarps + w) * run;
  if (rs64 >= rows) return;                  // warp-uniform
  const int rs = (int)rs64;
  const int nslab = min(run, rows - rs) / kSub;
  const bool draws = j < cols;
  // data role: pass it covers columns j0 + 4 it + lane / 8, rows (lane % 8) * 8 .. + 7 of the slab
  const int dc = lane >> 3, dr = (lane & 7) * 8;
  const int64_t col_stride = rows;
  const int64_t d0 = (int64_t)(j0 + dc) * col_stride + rs + dr;
  const int valid_cols = min(kTileCols, cols - j0);
  uint64_t* mb = reinterpret_cast<uint64_t*>(mask_out + (int64_t)j * (rows >> 3) + (rs >> 3));
  SlabPart<TI> cur;
  const bool full_group = valid_cols == kTileCols;
  if (full_group) cur.load(in + d0, col_stride, true);
  Xs128 s{0u, 0u, 0u, 1u};
  if (draws) s = start_state(st_in, cols, j, rs, tab);
#pragma unroll 1
  for (int q = 0; q < nslab; ++q) {
    SlabPart<TI> nxt;
    if (sizeof(TI) == 2 && full_group && q + 1 < nslab) nxt.load(in + d0 + (q + 1) * kSub, col_stride, true);
    uint64_t bits = 0;
    if (draws) bits = draw_keep64(s, thr24, kSub);
    const uint32_t lo = (uint32_t)bits, hi = (uint32_t)(bits >> 32);
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int c = 4 * it + dc;                       // column (within the group) this lane moves
      const uint32_t wl = __shfl_sync(0xffffffffu, lo, c), wh = __shfl_sync(0xffffffffu, hi, c);
      const uint32_t byte = ((dr < 32 ? wl : wh) >> (dr & 31)) & 0xFFu;
      if (c < valid_cols) {
        float x[8];
        if (full_group) {
          cur.get(it, x);
        } else {  // ragged last column group: this lane's 8 values directly
          const TI* src = in + d0 + (int64_t)4 * it * col_stride + q * kSub;
          if constexpr (sizeof(TI) == 2) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(src));
            const uint32_t ww[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              x[2 * e] = __uint_as_float(ww[e] << 16);
              x[2 * e + 1] = __uint_as_float(ww[e] & 0xFFFF0000u);
            }
          } else {
            const float4 a = __ldg(reinterpret_cast<const float4*>(src)), b = __ldg(reinterpret_cast<const float4*>(src) + 1);
            x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
          }
        }
        float r[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) r[e] = ((byte >> e) & 1u) ? __fmul_rn(x[e], scale) : 0.0f;
        store8_vec<TO>(out + d0 + (int64_t)4 * it * col_stride + q * kSub, r);
      }
    }
    if (draws) mb[q] = bits;
    if (full_group && q + 1 < nslab) {
      if (sizeof(TI) == 2) cur = nxt;                      // BF16: loaded one slab ahead
      else cur.load(in + d0 + (q + 1) * kSub, col_stride, true);
    }
  }
  if (draws && rs + nslab * kSub == rows) {  // this thread drew the column's last row
    st_out[j] = s.x;
    st_out[cols + j] = s.y;
    st_out[2 * cols + j] = s.z;
    st_out[3 * cols + j] = s.w;
  }
}

// Two streams at once: the xorshift chain of one stream is latency-bound
// (each step waits on the previous w), so a lane advances two independent
// row runs of its column with the steps interleaved.
__device__ __forceinline__ void draw_keep64x2(Xs128& a, Xs128& b, uint32_t thr24, uint64_t& ra, uint64_t& rb) {
  if (thr24 >= (1u << 24) || thr24 == 0) {
    ra = draw_keep64(a, thr24, kSub);
    rb = draw_keep64(b, thr24, kSub);
    return;
  }
  const uint32_t nthr = 0u - (thr24 << 8);
  uint32_t h[4];
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    uint32_t la = 0, lb = 0;
#pragma unroll kDrawUnroll
    for (int i = 0; i < 32; ++i) {
      const uint32_t wa = xs_step_fast(a), wb = xs_step_fast(b);
      asm("{ .reg .u32 d; add.cc.u32 d, %1, %2; addc.u32 %0, %0, %0; }" : "+r"(la) : "r"(wa), "r"(nthr));
      asm("{ .reg .u32 d; add.cc.u32 d, %1, %2; addc.u32 %0, %0, %0; }" : "+r"(lb) : "r"(wb), "r"(nthr));
    }
    h[2 * half] = __brev(la);
    h[2 * half + 1] = __brev(lb);
  }
  ra = (uint64_t)h[0] | ((uint64_t)h[2] << 32);
  rb = (uint64_t)h[1] | ((uint64_t)h[3] << 32);
}

template <typename TO, int N>
__device__ __forceinline__ void store_vec_n(TO* op, const float (&r)[N]) {
  if constexpr (sizeof(TO) == 2) {
    uint32_t u[N / 2];
    pack_bf16_ref_n<N / 2>(r, u);
    if constexpr (N == 8) *reinterpret_cast<uint4*>(op) = make_uint4(u[0], u[1], u[2], u[3]);
    else *reinterpret_cast<uint2*>(op) = make_uint2(u[0], u[1]);
  } else {
#pragma unroll
    for (int q = 0; q < N / 4; ++q)
      reinterpret_cast<float4*>(op)[q] = make_float4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
  }
}

// Four streams at once (see draw_keep64x2).
__device__ __forceinline__ void draw_keep64x4(Xs128 (&s)[4], uint32_t nthr, uint64_t (&r)[4]) {
  uint32_t h[2][4];
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    uint32_t l[4] = {0u, 0u, 0u, 0u};
#pragma unroll kDrawUnroll
    for (int i = 0; i < 32; ++i) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t w = xs_step_fast(s[q]);
        asm("{ .reg .u32 d; add.cc.u32 d, %1, %2; addc.u32 %0, %0, %0; }" : "+r"(l[q]) : "r"(w), "r"(nthr));
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) h[hf][q] = __brev(l[q]);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) r[q] = (uint64_t)h[0][q] | ((uint64_t)h[1][q] << 32);
}

// DROPOUT fused, TMA-fed (dense column-major BF16 / FP32 views, rows % 64
// == 0).  Warp = 32 consecutive columns x one run of `run` rows split into NS
// equal parts (NS = 4 for BF16 input, 2 for FP32; each part a power-of-two
// multiple of 64 rows) that the lanes draw as NS interleaved streams -- the
// xorshift chain is latency-bound, so the interleave is the ILP (lane =
// column; part 0 jumps from the seed by popcount(run index) levels, the
// others are one or two jumps from it).  The warp's 32 x 64-row input slabs
// arrive by TMA into a private kStages-deep shared-memory ring (the HBM reads
// stay in flight without holding registers), in the order (slab 0 of parts
// 0..NS-1), (slab 1 ...), ...; per slab each lane takes 16-byte chunks (8 or
// 16 lanes per column: conflict-free), fetches the chunk's keep bits from the
// drawing lane with a shuffle, applies keep ? x * scale : 0 (DROPOUT_INV's
// rule, FP32 math; RNE + the reference NaN rule for BF16 out) and stores
// coalesced; the drawing lane stores the slab's 8-byte mask word.  Bitwise
// the same draws, mask and values as the other DROPOUT paths (ops.py:430-444).
constexpr int kDropWarps = 4;
template <typename TI> struct DropTma {
  static constexpr int kStreams = sizeof(TI) == 2 ? TPP_DROP_NS : 2;
  static constexpr int kStages = sizeof(TI) == 2 ? TPP_DROP_STAGES : 3;
  static constexpr int kSlab = 32 * kSub * (int)sizeof(TI);  // bytes per warp slab
  static constexpr int kSmem = kDropWarps * kStages * kSlab + kDropWarps * kStages * 8;
};

template <typename TI, typename TO>
__global__ void __launch_bounds__(kDropWarps * 32) dropout_tma_kernel(
    const __grid_constant__ CUtensorMap tin, const uint32_t* __restrict__ st_in, uint32_t* __restrict__ st_out,
    uint32_t thr24, TO* __restrict__ out, int64_t out_ld, uint8_t* __restrict__ mask_out, int rows, int cols,
    int run, float scale, const uint4* __restrict__ tab) {
  using namespace sm100;
  constexpr int E = sizeof(TI), S = DropTma<TI>::kStages, SLAB = DropTma<TI>::kSlab, NS = DropTma<TI>::kStreams;
  constexpr int EPC = 16 / E;      // elements per 16-byte chunk
  constexpr int CPC = kSub / EPC;  // chunks per column of a slab (= passes per slab)
  extern __shared__ __align__(128) uint8_t dsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // item = (column group, row run), flattened so the grid fits one wave
  const int64_t item = (int64_t)blockIdx.x * kDropWarps + w;
  const int segs = (rows + run - 1) / run;
  const int64_t cg = item / segs;
  if (cg * 32 >= cols) return;  // warp-uniform; barriers and ring are private to the warp
  const int rs = (int)(item - cg * segs) * run, part = run / NS;
  uint8_t* ring = dsm + (size_t)w * S * SLAB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(dsm + (size_t)kDropWarps * S * SLAB) + w * S;
  const int j0 = (int)cg * 32, j = j0 + lane;
  int n[NS];  // slabs per stream (non-increasing)
#pragma unroll
  for (int i = 0; i < NS; ++i) n[i] = max(0, min(part, rows - rs - i * part)) / kSub;
  // TMA producer cursor (lane 0): slab q of stream i, streams inner
  int pq = 0, pi = 0, issued = 0;
  auto issue_next = [&]() {
    const int st = issued % S;
    mbar_arrive_expect_tx(&bars[st], SLAB);
    tma_load_5d(ring + st * SLAB, &tin, &bars[st], (rs + pi * part + pq * kSub) * E / 2, j0, 0, 0, 0);
    ++issued;
    ++pi;
    int npi = 0;  // n[pi] without dynamic indexing (keeps n in registers)
#pragma unroll
    for (int i = 1; i < NS; ++i) npi = pi == i ? n[i] : npi;
    if (pi == NS || pq >= npi) pi = 0, ++pq;
  };
  int total = 0;
#pragma unroll
  for (int i = 0; i < NS; ++i) total += n[i];
  if (lane == 0) {
    for (int st = 0; st < S; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
    while (issued < min(S, total)) issue_next();
  }
  __syncwarp();
  const bool draws = j < cols;
  const int valid_cols = min(32, cols - j0);
  Xs128 sv[NS];
  {
    const int lp = 31 - __clz(part / kSub);  // jump level of one part
    sv[0] = draws ? start_state(st_in, cols, j, rs, tab) : Xs128{0u, 0u, 0u, 1u};
    if constexpr (NS == 2) {
      sv[1] = n[1] > 0 && draws ? jump(sv[0], tab + lp * kNibs * 16) : sv[0];
    } else {
      sv[1] = n[1] > 0 && draws ? jump(sv[0], tab + lp * kNibs * 16) : sv[0];
      sv[2] = n[2] > 0 && draws ? jump(sv[0], tab + (lp + 1) * kNibs * 16) : sv[0];
      sv[3] = n[3] > 0 && draws ? jump(sv[2], tab + lp * kNibs * 16) : sv[0];
    }
  }
  uint8_t* mcol = mask_out + (int64_t)j * (rows >> 3);
  // apply-phase mapping: pass p, lane -> column p * CPP + lane / CPC of the
  // group, rows b0 .. b0 + EPC - 1 of the slab (b0 fixed per lane)
  constexpr int CPP = 32 / CPC;  // columns per pass
  const int lane_c = lane / CPC, b0 = (lane % CPC) * EPC;
  const int lane_smem = lane_c * kSub * E + (lane % CPC) * 16;
  TO* const obase = out + (int64_t)(j0 + lane_c) * out_ld + b0;
  const int64_t ostride = (int64_t)CPP * out_ld;
  const bool special = thr24 >= (1u << 24) || thr24 == 0;
  int k = 0;
#pragma unroll 1
  for (int q = 0; q < n[0]; ++q) {
    uint64_t bw[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) bw[i] = 0ull;
    if (draws) {
      if (!special && q < n[NS - 1]) {
        if constexpr (NS == 4) draw_keep64x4(sv, 0u - (thr24 << 8), bw);
        else draw_keep64x2(sv[0], sv[1], thr24, bw[0], bw[1]);
      } else {
#pragma unroll
        for (int i = 0; i < NS; ++i)
          if (q < n[i]) bw[i] = draw_keep64(sv[i], thr24, kSub);
      }
    }
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      if (q >= n[i]) break;  // n is non-increasing
      const uint64_t bits = bw[i];
      const int row0 = rs + i * part + q * kSub;
      const int st = k % S;
      mbar_wait(&bars[st], (uint32_t)(k / S) & 1u);
      const uint8_t* sl = ring + st * SLAB + lane_smem;
      TO* o = obase + row0;
      const uint32_t lo = (uint32_t)bits, hi = (uint32_t)(bits >> 32);
#pragma unroll
      for (int pass = 0; pass < CPC; ++pass) {
        const int c = pass * CPP + lane_c;  // column (within the group) of this lane's chunk
        const uint32_t wl = __shfl_sync(0xffffffffu, lo, c), wh = __shfl_sync(0xffffffffu, hi, c);
        const uint32_t kb = ((b0 < 32 ? wl : wh) >> (b0 & 31)) & ((1u << EPC) - 1u);
        if (c < valid_cols) {
          const uint4 v = *reinterpret_cast<const uint4*>(sl + pass * CPP * kSub * E);
          float x[EPC];
          if constexpr (E == 2) {
            const uint32_t ww[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              x[2 * e] = __uint_as_float(ww[e] << 16);
              x[2 * e + 1] = __uint_as_float(ww[e] & 0xFFFF0000u);
            }
          } else {
            x[0] = __uint_as_float(v.x); x[1] = __uint_as_float(v.y);
            x[2] = __uint_as_float(v.z); x[3] = __uint_as_float(v.w);
          }
          float r[EPC];
#pragma unroll
          for (int e = 0; e < EPC; ++e) r[e] = ((kb >> e) & 1u) ? __fmul_rn(x[e], scale) : 0.0f;
          store_vec_n<TO, EPC>(o + pass * ostride, r);
        }
      }
      if (draws) *reinterpret_cast<uint64_t*>(mcol + (row0 >> 3)) = bits;
      __syncwarp();  // every lane's reads of this stage are done before TMA refills it
      if (lane == 0 && issued < total) issue_next();
      ++k;
    }
  }
  if (draws) {  // the stream that drew the column's last row hands the state on
    bool last = false;
    Xs128 f = sv[0];
#pragma unroll
    for (int i = 0; i < NS; ++i)
      if (n[i] > 0 && rs + i * part + n[i] * kSub == rows) last = true, f = sv[i];
    if (last) {
      st_out[j] = f.x;
      st_out[cols + j] = f.y;
      st_out[2 * cols + j] = f.z;
      st_out[3 * cols + j] = f.w;
    }
  }
}

template <typename TI, typename TO>
static int launch_dropout_tma(const CUtensorMap& m, const uint32_t* st_in, uint32_t* st_out, uint32_t thr24, void* out,
                              int64_t out_ld, uint8_t* mask_out, int rows, int cols, int run, float scale,
                              const uint4* tab, dim3 grid, cudaStream_t s) {
  constexpr int smem = DropTma<TI>::kSmem;
  cudaError_t e = ensure_smem_attr((const void*)dropout_tma_kernel<TI, TO>, smem);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(dropout_tma_kernel)");
  dropout_tma_kernel<TI, TO><<<grid, kDropWarps * 32, smem, s>>>(m, st_in, st_out, thr24, reinterpret_cast<TO*>(out),
                                                                  out_ld, mask_out, rows, cols, run, scale, tab);
  TPP_CUDA_LAUNCH_CHECK("dropout_tma_kernel");
  return TPP_OK;
}

// PRNG fill (ops.py:416-427): FP32 uniforms.  Item = blockIdx.x: column group
// item / parts, row part item % parts; warp w draws `run` contiguous rows, 64
// at a time into shared memory, and the CTA streams each 32 x (8 x 64) slab.
__global__ void __launch_bounds__(256) prng_fill_kernel(const uint32_t* __restrict__ st_in,
                                                        uint32_t* __restrict__ st_out, float* out, int out_ld,
                                                        int rows, int cols, int run, int parts, int vec,
                                                        const uint4* __restrict__ tab) {
  extern __shared__ float fill[];  // [32][kFillStride]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cg = blockIdx.x / parts, part = blockIdx.x - cg * parts;
  const int c0 = cg * kTileCols, j = c0 + lane;
  const int base = part * run * kWarps;  // first row of the item
  const int rs = base + w * run;         // first row of this thread's run
  const int nr = max(0, min(run, rows - rs));
  const bool active = j < cols && nr > 0;
  Xs128 s{0, 0, 0, 0};
  if (active) s = start_state(st_in, cols, j, rs, tab);
#pragma unroll 1
  for (int q = 0; q < run / kSub; ++q) {
    const int n = active ? max(0, min(kSub, nr - q * kSub)) : 0;
    for (int i = 0; i < n; ++i)
      fill[lane * kFillStride + w * kSub + i] = (float)(xs_step(s) >> 8) * 5.9604644775390625e-08f;
    __syncthreads();
#pragma unroll 2
    for (int idx = threadIdx.x; idx < kTileCols * kWarps * (kSub / 8); idx += 256) {
      const int cc = idx >> 6, piece = (idx >> 3) & 7, gq = idx & 7;
      const int row = base + piece * run + q * kSub + gq * 8;
      if (row >= rows || c0 + cc >= cols) continue;
      float r[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) r[e] = fill[cc * kFillStride + piece * kSub + gq * 8 + e];
      store8<float>(out, TPP_FP32, out_ld, row, c0 + cc, rows, vec && row + 8 <= rows, r);
    }
    __syncthreads();
  }
  if (active && rs + nr == rows) {
    st_out[j] = s.x;
    st_out[cols + j] = s.y;
    st_out[2 * cols + j] = s.z;
    st_out[3 * cols + j] = s.w;
  }
}

// DROPOUT_INV (ops.py:378-382): one thread per mask byte (8 rows of a column).
template <typename T, typename I>
__global__ void dropout_inv_kernel(DView in, const uint8_t* __restrict__ mask, T scale, void* out,
                                   int out_dtype, int out_ld, int vec) {
  const int rows = in.rows;
  const I bpc = (I)((rows + 7) >> 3);
  const I groups = bpc * (I)in.cols;
  constexpr int kU = 4;
  for (I base = blockIdx.x * (I)blockDim.x + threadIdx.x; base < groups; base += (I)gridDim.x * blockDim.x * kU) {
    T x[kU][8];
    I g[kU];
    int j[kU], i0[kU];
    uint32_t mb[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      g[u] = base + (I)u * gridDim.x * blockDim.x;
      j[u] = (int)(g[u] / bpc);
      i0[u] = (int)(g[u] - (I)j[u] * bpc) * 8;
      mb[u] = g[u] < groups ? mask[g[u]] : 0u;
      if (g[u] < groups) load8<T>(in, i0[u], j[u], rows, vec && i0[u] + 8 <= rows, x[u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (g[u] >= groups) continue;
      scale8<T>(mb[u], scale, x[u]);
      store8<T>(out, out_dtype, out_ld, i0[u], j[u], rows, vec && i0[u] + 8 <= rows, x[u]);
    }
  }
}

static bool vec_ok(const DView& in, const void* out, int out_dtype, int out_ld, bool f64) {
  if (f64) return false;
  const bool in_ok = in.bcast == TPP_BCAST_NONE && (in.dtype == TPP_FP32 || in.dtype == TPP_BF16) &&
                     (in.ld & 7) == 0 && ((uintptr_t)in.p & 15) == 0;
  const bool out_ok = (out_dtype == TPP_FP32 || out_dtype == TPP_BF16) && (out_ld & 7) == 0 &&
                      ((uintptr_t)out & 15) == 0;
  return in_ok && out_ok;
}

}  // namespace

int launch_prng_seed(uint64_t seed, int cols, uint32_t* state, cudaStream_t s) {
  int rc = TPP_OK;
  if (!jump_tables(&rc)) return rc;
  prng_seed_kernel<<<(cols + 255) / 256, 256, 0, s>>>(seed, cols, state);
  TPP_CUDA_LAUNCH_CHECK("prng_seed_kernel");
  return TPP_OK;
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

static bool dropout_unfused() {  // experiments: TPP_DROPOUT_UNFUSED=1 keeps mask kernel + DROPOUT_INV
  static const bool v = getenv("TPP_DROPOUT_UNFUSED") != nullptr;
  return v;
}

int launch_prng_tile(int mode, const DView& in, const uint32_t* st_in, uint32_t* st_out, double p,
                     void* out, int out_dtype, int out_ld, uint8_t* mask_out, int rows, int cols, bool f64,
                     cudaStream_t s) {
  int rc = TPP_OK;
  const uint4* tab = jump_tables(&rc);
  if (!tab) return rc;
  if (rows > (1 << 30)) return TPP_E_UNSUPPORTED;
  const int64_t cgroups = (cols + kTileCols - 1) / kTileCols;
  if (mode == 0) {
    // ~3 items per SM; each warp's run a multiple of 64 rows
    const int64_t max_parts = ((int64_t)rows + kSub * kWarps - 1) / (kSub * kWarps);
    int64_t parts = (3 * (int64_t)sm_count() + cgroups - 1) / cgroups;
    parts = parts < 1 ? 1 : (parts > max_parts ? max_parts : parts);
    const int64_t per_part = ((int64_t)rows + parts - 1) / parts;
    const int run = (int)(((per_part + kWarps - 1) / kWarps + kSub - 1) / kSub * kSub);
    parts = ((int64_t)rows + (int64_t)run * kWarps - 1) / ((int64_t)run * kWarps);
    if (cgroups * parts > 0x7fffffff) return TPP_E_UNSUPPORTED;
    const int smem = kTileCols * kFillStride * (int)sizeof(float);
    {
      cudaError_t e = ensure_smem_attr((const void*)prng_fill_kernel, smem);
      if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(prng_fill_kernel)");
    }
    const int vec = (out_ld & 7) == 0 && ((uintptr_t)out & 15) == 0;
    prng_fill_kernel<<<(unsigned)(cgroups * parts), kWarps * 32, smem, s>>>(
        st_in, st_out, reinterpret_cast<float*>(out), out_ld, rows, cols, run, (int)parts, vec, tab);
    TPP_CUDA_LAUNCH_CHECK("prng_fill_kernel");
    return TPP_OK;
  }
  // 1) keep mask.  keep <=> (float)(w >> 8) * 2^-24 >= float32(p) <=> (w >> 8) >= ceil(float32(p) * 2^24)
  const double thr = std::ceil((double)(float)p * 16777216.0);
  const uint32_t thr24 = (uint32_t)thr;  // <= 2^24; 2^24 means "never keep"
  // TPP_DROPOUT_FUSED=2: the register-staged fused kernel below instead of
  // the TMA-fed one (experiments)
  static const int fused_mode = [] {
    const char* e = getenv("TPP_DROPOUT_FUSED");
    return e ? atoi(e) : 0;
  }();
  // dense column-major BF16 / FP32 views with whole 64-row slabs: draws and
  // the scaled copy fused into one pass -- TMA-fed (dropout_tma_kernel)
  static const bool no_tma = fused_mode == 2;  // experiments
  const int esz = in.dtype == TPP_BF16 ? 2 : 4;
  if (!f64 && !no_tma && rows % kSub == 0 && in.bcast == TPP_BCAST_NONE &&
      (in.dtype == TPP_BF16 || in.dtype == TPP_FP32) && (out_dtype == TPP_BF16 || out_dtype == TPP_FP32) &&
      ((uintptr_t)in.p & 15) == 0 && ((int64_t)in.ld * esz) % 16 == 0 && in.ld >= rows &&
      ((uintptr_t)out & 15) == 0 && out_ld >= rows && out_ld % 8 == 0 && ((uintptr_t)mask_out & 7) == 0 &&
      !dropout_unfused()) {
    // CTAs resident per SM (the shared-memory ring bounds it)
    const int per_sm = std::max(1, (227 * 1024) / (esz == 2 ? DropTma<uint16_t>::kSmem : DropTma<float>::kSmem));
    const int64_t warps = (int64_t)sm_count() * per_sm * kDropWarps;
    // run: the smallest power-of-two multiple of (streams x 64) rows whose items fit one wave
    int64_t run64 = (esz == 2 ? DropTma<uint16_t>::kStreams : DropTma<float>::kStreams) * kSub;
    while (cgroups * (((int64_t)rows + run64 - 1) / run64) > warps && run64 < rows) run64 *= 2;
    const int run = (int)run64;
    const int64_t segs = ((int64_t)rows + run - 1) / run;
    const int64_t ctas = (cgroups * segs + kDropWarps - 1) / kDropWarps;
    if (ctas <= 0x7fffffff) {
      CUtensorMap m;
      const uint64_t dims[5] = {(uint64_t)rows * esz / 2, (uint64_t)cols, 1, 1, 1};
      const uint64_t str[4] = {(uint64_t)in.ld * esz, (uint64_t)in.ld * esz * cols, (uint64_t)in.ld * esz * cols,
                               (uint64_t)in.ld * esz * cols};
      const uint32_t box[5] = {(uint32_t)(kSub * esz / 2), 32, 1, 1, 1};
      int mrc = make_tma_map_5d(&m, in.p, dims, str, box, 0);
      if (mrc != TPP_OK) return mrc;
      const float scale = compute_scale<float>(p);
      const dim3 grid((unsigned)ctas);
      if (in.dtype == TPP_BF16 && out_dtype == TPP_BF16)
        return launch_dropout_tma<uint16_t, uint16_t>(m, st_in, st_out, thr24, out, out_ld, mask_out, rows, cols, run,
                                                      scale, tab, grid, s);
      if (in.dtype == TPP_BF16)
        return launch_dropout_tma<uint16_t, float>(m, st_in, st_out, thr24, out, out_ld, mask_out, rows, cols, run,
                                                   scale, tab, grid, s);
      if (out_dtype == TPP_BF16)
        return launch_dropout_tma<float, uint16_t>(m, st_in, st_out, thr24, out, out_ld, mask_out, rows, cols, run,
                                                   scale, tab, grid, s);
      return launch_dropout_tma<float, float>(m, st_in, st_out, thr24, out, out_ld, mask_out, rows, cols, run, scale,
                                              tab, grid, s);
    }
  }
  if (!f64 && rows % kSub == 0 && in.ld == rows && out_ld == rows && in.bcast == TPP_BCAST_NONE &&
      (in.dtype == TPP_BF16 || in.dtype == TPP_FP32) && (out_dtype == TPP_BF16 || out_dtype == TPP_FP32) &&
      ((uintptr_t)in.p & 15) == 0 && ((uintptr_t)out & 15) == 0 && ((uintptr_t)mask_out & 7) == 0 &&
      !dropout_unfused()) {
    const int64_t target_threads = (int64_t)sm_count() * 1024;
    int64_t run64 = ((int64_t)rows * cols + target_threads - 1) / target_threads;
    run64 = (run64 + kSub - 1) / kSub * kSub;
    if (run64 < kSub) run64 = kSub;
    if (run64 > rows) run64 = rows;
    const int run = (int)run64;
    const int64_t segs = ((int64_t)rows + run - 1) / run;
    const int64_t gy = (segs + kWarps - 1) / kWarps;
    if (gy <= 65535 && cgroups <= 0x7fffffff) {
      const float scale = compute_scale<float>(p);
      const dim3 grid((unsigned)cgroups, (unsigned)gy);
      if (in.dtype == TPP_BF16 && out_dtype == TPP_BF16)
        dropout_fused_kernel<uint16_t, uint16_t><<<grid, kWarps * 32, 0, s>>>(
            st_in, st_out, thr24, (const uint16_t*)in.p, (uint16_t*)out, mask_out, rows, cols, run, scale, tab);
      else if (in.dtype == TPP_BF16)
        dropout_fused_kernel<uint16_t, float><<<grid, kWarps * 32, 0, s>>>(
            st_in, st_out, thr24, (const uint16_t*)in.p, (float*)out, mask_out, rows, cols, run, scale, tab);
      else if (out_dtype == TPP_BF16)
        dropout_fused_kernel<float, uint16_t><<<grid, kWarps * 32, 0, s>>>(
            st_in, st_out, thr24, (const float*)in.p, (uint16_t*)out, mask_out, rows, cols, run, scale, tab);
      else
        dropout_fused_kernel<float, float><<<grid, kWarps * 32, 0, s>>>(
            st_in, st_out, thr24, (const float*)in.p, (float*)out, mask_out, rows, cols, run, scale, tab);
      TPP_CUDA_LAUNCH_CHECK("dropout_fused_kernel");
      return TPP_OK;
    }
  }
  // runs sized for ~32 resident warps per SM (a jump costs ~32 L1 loads)
  const int64_t target_threads = (int64_t)sm_count() * 1024;
  int64_t run64 = ((int64_t)rows * cols + target_threads - 1) / target_threads;
  run64 = (run64 + kSub - 1) / kSub * kSub;
  const int64_t rows64 = ((int64_t)rows + kSub - 1) / kSub * kSub;
  if (run64 < kSub) run64 = kSub;
  if (run64 > rows64) run64 = rows64;
  const int run = (int)run64;
  const int64_t segs = ((int64_t)rows + run - 1) / run;
  const int64_t gy = (segs + kWarps - 1) / kWarps;
  if (gy > 65535 || cgroups > 0x7fffffff) return TPP_E_UNSUPPORTED;
  const int mask8 = ((rows + 7) / 8) % 8 == 0 && ((uintptr_t)mask_out & 7) == 0;
  dropout_mask_kernel<<<dim3((unsigned)cgroups, (unsigned)gy), kWarps * 32, 0, s>>>(st_in, st_out, thr24, mask_out,
                                                                                 rows, cols, run, mask8, tab);
  TPP_CUDA_LAUNCH_CHECK("dropout_mask_kernel");
  // 2) out = keep ? x * compute_dtype(1 / (1 - p)) : 0
  return launch_dropout_inv(in, mask_out, p, out, out_dtype, out_ld, f64, s);
}

int launch_dropout_inv(const DView& in, const uint8_t* mask, double p, void* out, int out_dtype, int out_ld,
                       bool f64, cudaStream_t s) {
  const int64_t groups = (int64_t)((in.rows + 7) / 8) * in.cols;
  int64_t blocks = (groups + 1023) / 1024;
  if (blocks > 148 * 8) blocks = 148 * 8;
  const int vec = vec_ok(in, out, out_dtype, out_ld, f64);
  const bool small = groups < (1ll << 30);  // 32-bit index math
  if (f64) {
    const double sc = p < 1.0 ? compute_scale<double>(p) : 0.0;
    if (small)
      dropout_inv_kernel<double, uint32_t><<<(unsigned)blocks, 256, 0, s>>>(in, mask, sc, out, out_dtype, out_ld, vec);
    else
      dropout_inv_kernel<double, int64_t><<<(unsigned)blocks, 256, 0, s>>>(in, mask, sc, out, out_dtype, out_ld, vec);
  } else {
    const float sc = p < 1.0 ? compute_scale<float>(p) : 0.f;
    const int rc = fast_dropout_inv(in, mask, sc, out, out_dtype, out_ld, s);
    if (rc == 0) return TPP_OK;
    if (rc == 2) return cuda_status(cudaGetLastError(), "dropout_inv_vec_kernel");
    if (small)
      dropout_inv_kernel<float, uint32_t><<<(unsigned)blocks, 256, 0, s>>>(in, mask, sc, out, out_dtype, out_ld, vec);
    else
      dropout_inv_kernel<float, int64_t><<<(unsigned)blocks, 256, 0, s>>>(in, mask, sc, out, out_dtype, out_ld, vec);
  }
  TPP_CUDA_LAUNCH_CHECK("dropout_inv_kernel");
  return TPP_OK;
}

}  // namespace tpp

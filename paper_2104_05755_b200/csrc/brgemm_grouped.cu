// K11: the BRGEMM TPP itself on tcgen05 — brgemm() over STRIDE / OFFSET /
// ADDRESS batches of arbitrary BF16 blocks, many C blocks per launch.
//
// Reference semantics (contraction.py:261-322): for every group g (one C
// block; a single brgemm() call is one group)
//     C_g = beta * C_g + sum_i A_{g,i} x B_{g,i}
// with A_{g,i} an m x k block (PLAIN column-major with lda, or VNNI-2
// [ceil(k/2)][m][2], contraction.py:238-247), B_{g,i} a k x n column-major
// block (ldb), C an m x n FP32 column-major block (ldc).  The blocks live at
// arbitrary (16-byte aligned) addresses — the batch is an address / offset /
// stride list, not a tensor — so operands cannot come through a TMA tensor
// map.  Instead 8 producer warps move each (entry i, 64-deep k chunk) stage
// from global memory straight into the UMMA-canonical 128B-swizzled smem
// layouts:
//   B        K-major (k contiguous per column): 16-byte cp.async per chunk
//   A PLAIN  MN-major (m contiguous per k):     16-byte cp.async per chunk
//   A VNNI   K-major: 4 x 16-byte cp.async of (4 k-pairs x 4 rows) into a raw
//            area, then a 32-bit word transpose into 4 x 16-byte row chunks
// (zero fill past m, n, k), STAGES - 2 stages in flight per thread (cp.async
// groups; VNNI A lands raw and each thread transposes its own words once its
// group completed), then fence.proxy.async and an mbarrier arrive hand the
// stage to the MMA warp.  The MMA warp issues
// tcgen05.mma kind::f16 (M = 64 when the C block has <= 64 rows, else 128;
// N = 64/128/256) into a double-buffered TMEM accumulator — the whole batch
// of a tile accumulates on chip — and 4 epilogue warps apply beta and store
// FP32 C (coalesced: a warp writes 32 consecutive rows of a column).
//
// Persistent CTAs walk work items (group, row tile, column tile).

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "sm100.cuh"
#include "launch.h"

namespace tpp {
using namespace sm100;
namespace grp {

constexpr int kEpiWarps = 4;    // warps 0-3: epilogue (TMEM lane quarter = warp)
constexpr int kProdWarp0 = 4;   // warps 4-7: issue the stage copies, never wait for data
constexpr int kProdWarps = 4;
constexpr int kProd = 32 * kProdWarps;
constexpr int kFinWarp0 = kProdWarp0 + kProdWarps;  // warps 8-11: land a stage (VNNI transpose, proxy fence)
constexpr int kFinWarps = 4;
constexpr int kMmaWarp = kFinWarp0 + kFinWarps;     // MMA issue + TMEM allocation
constexpr int kThreads = 32 * (kMmaWarp + 1);

struct GParams {
  int m, n, k, lda, ldb, ldc;
  int vnni;         // A layout: 0 PLAIN, 1 VNNI-2
  int kind;         // 0 STRIDE, 1 OFFSET, 2 ADDRESS
  const uint16_t* a;
  const uint16_t* b;
  long long stride_a, stride_b;
  const long long* a_idx;  // STRIDE: per-group offsets [groups] (or null); OFFSET: [groups*count]; ADDRESS: pointers
  const long long* b_idx;
  long long count;
  float* c;
  const long long* c_off;  // per-group C offsets (elements) or null (one group)
  long long groups;
  int tiles_m, tiles_n, kchunks;
  int dims_ok;      // m, k, ldb (lda for PLAIN A) multiples of 8: 16-byte chunks never straddle an edge
  float beta;
  int beta_mode;    // 0: beta == 0, 1: beta == 1, 2: general
  int dbg;          // experiments (TPP_GRP_DBG): 1 no MMAs, 2 no copies, 4 no VNNI transpose
  // Gangs (optional): a work item is gang_ma x gang_nb groups that share A
  // lists along a row and B lists along a column (the reference's FC / conv
  // compositions: every C block of one weight block row reuses its A blocks).
  // A rows of sub-block ma come from group gang_rows[j][ma], B rows of
  // sub-block nb from gang_cols[j][nb], C of (ma, nb) is group
  // gang_cells[j][ma][nb]; -1 = empty (zero operands, no store).  Sub-blocks:
  // 64 rows of A (m <= 64) and, when gang_nb > 1, 64 rows of B (n <= 64).
  int gang_ma, gang_nb, ngangs;
  const int* gang_rows;
  const int* gang_cols;
  const int* gang_cells;
  long long* trace;   // TPP_GRP_TRACE: CTA 0's clock64 stamps per stage (probe only)
  // TMA staging (STRIDE / OFFSET batches, power-of-two row pitches): a stage
  // whose blocks all start on a row of the tensor maps' 2-D views is loaded
  // by one thread's TMA boxes instead of 12+ cp.async per producer thread
  int tma;
  int a_shift, b_shift;   // log2 of the A row pitch (VNNI: 2m, PLAIN: lda) and of ldb, in elements
  int b_box;              // B rows per box (a B sub-block or the whole BN tile)
  int a_rbits, b_rbits;   // log2 of the views' row counts
  // BF16 output (beta = 0): C emitted RNE-narrowed (dtypes.py:82-97) at
  // c16 + c_off, block column v -> column (v / col_period) * col_keep +
  // v % col_period, dropped when v % col_period >= col_keep (the conv
  // composition's padded-width rows; col_period = n keeps all)
  uint16_t* c16;
  int col_period, col_keep;
  unsigned col_magic;   // ceil(2^32 / col_period): v / col_period = umulhi(v, magic) for the block's columns
  // VNNI A through tensor memory (M = 128, TMA mode): a VNNI word (row m,
  // k pair) is exactly a TMEM cell of the MMA's A operand (lane m, one column
  // per k pair), so the finisher copies raw words smem -> TMEM (tcgen05.st)
  // instead of transposing them into a K-major smem tile
  int tmem_a;
};
constexpr int kTrace = 128;   // stages traced
constexpr int kGangMA = 2, kGangNB = 4;

constexpr int kIdxChunk = 256;  // batch entries whose indices sit in smem at a time
constexpr int kTmaRowBits = 30;  // rows of the TMA maps' 2-D views of a / b (at most; strides stay < 2^39 B)

// TA: VNNI A through tensor memory -- no K-major A tile in the stage, so
// deeper rings fit
template <int BM, int BN, int STAGES, bool TA = false>
struct GSmem {
  static constexpr int A_BYTES = TA ? 0 : BM * 128;  // BM rows x 64 k (bf16)
  static constexpr int B_BYTES = BN * 128;
  static constexpr int RAW_BYTES = BM * 128;  // VNNI A as loaded, before the word transpose
  static constexpr int STAGE = A_BYTES + B_BYTES + RAW_BYTES;
  static constexpr int IDX_OFF = STAGES * STAGE;                 // batch index chunk [slots][kIdxChunk]
  static constexpr int BAR_OFF = IDX_OFF + (kGangMA + kGangNB) * kIdxChunk * 8;
  static constexpr int BYTES = BAR_OFF + (3 * STAGES + 4) * 8 + 16 + 1024;
  static constexpr int TMEM_COLS = 2 * BN;
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint4 ldg_nc16(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
// explicit shared-space accesses: the aligned dynamic smem pointer is an
// integer round trip, so plain C++ accesses through it compile to GENERIC
// loads -- six dependent ones per stage cost the producers ~700 cycles
__device__ __forceinline__ long long lds64(uint32_t a) {
  long long v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, long long v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void sts16(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint32_t selp32(uint32_t a, uint32_t b, int c) {   // c ? a : b, no branch
  uint32_t r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\tselp.b32 %0, %1, %2, q;\n\t}" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
// v rotated left by rot (0..3) words: result word j = v word (j + rot) & 3
__device__ __forceinline__ uint4 rot4(uint4 v, int rot) {
  const int r1 = rot & 1, r2 = rot & 2;
  uint4 t = make_uint4(selp32(v.y, v.x, r1), selp32(v.z, v.y, r1), selp32(v.w, v.z, r1), selp32(v.x, v.w, r1));
  return make_uint4(selp32(t.z, t.x, r2), selp32(t.w, t.y, r2), selp32(t.x, t.z, r2), selp32(t.y, t.w, r2));
}

// the producer's walk over (work item, batch entry, k chunk)
struct StageIt {
  int tile;
  long long i;
  int kc;
};

template <int BM, int BN, int STAGES, bool TA>
__global__ void __launch_bounds__(kThreads, 1)
    brgemm_grouped_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const GParams p) {
  using S = GSmem<BM, BN, STAGES, TA>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* landed = tempty + 2;   // a stage's copies are in smem (issue warps -> finisher warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(landed + STAGES);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  // work items: gangs x column tiles, or groups x row tiles x column tiles (< 2^31, checked by the host)
  const int ntiles = p.gang_cells ? p.ngangs * p.tiles_n : (int)(p.groups * p.tiles_m * p.tiles_n);
  const long long per_tile = p.count * p.kchunks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], kFinWarps);   // one arrival per finisher warp
      mbar_init(&empty[s], 1);
      mbar_init(&landed[s], p.tma ? 1 : kProd);   // TMA mode: one arrival per stage (its issuing lane)
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);
    }
    fence_mbar_init();
  }
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) p.trace[7 * kTrace] = clock64();
  const uint32_t tcols = TA ? 512u : (uint32_t)S::TMEM_COLS;   // + STAGES x 32 A columns
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp >= kProdWarp0 && warp < kProdWarp0 + kProdWarps) {
    // ============================ producers ============================
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int t = threadIdx.x - kProdWarp0 * 32;
    // ---- per-thread chunk assignments, fixed for the whole kernel (the
    // fast path's per-stage work is then a few adds per 16-byte copy) ----
    // B (K-major, BN rows x 8 chunks): rows br0 + BRS j, chunk bq
    constexpr int BRS = kProd / 8, BJ = BN / BRS;
    const int br0 = t >> 3, bq = t & 7;
    const uint32_t b_soff = (br0 >> 3) * 1024 + (br0 & 7) * 128 + ((bq ^ (br0 & 7)) << 4);  // + j * BRS * 128
    // A PLAIN (MN-major, 64 k rows x BM/8 chunks): k rows akk0 + AKS j, chunk ach
    constexpr int CPR = BM / 8, AKS = kProd / CPR, AJ = 64 / AKS;
    const int akk0 = t / CPR, ach = t % CPR;
    const uint32_t a_soff = (ach >> 3) * 8192 + (akk0 >> 3) * 1024 + (akk0 & 7) * 128 +
                            (((ach & 7) ^ (akk0 & 7)) << 4);  // + j * AKS * 128
    // A VNNI: units (k-pair quad pq, row quad mq) = t + u * 128
    constexpr int AU = (BM * 2 + kProd - 1) / kProd;   // units of 4 k-pairs x 4 rows: 8 * BM / 4 in all
    constexpr int NUNITS = BM * 2;
    // raw VNNI A in smem, the TMA boxes' layout: [sub-block][k-pair 0..31][row]
    // of 32-bit words, a sub-block = 64 rows (gangs) or the whole tile
    const int bmsub = p.gang_ma == 2 ? 64 : BM;
    auto raw_off = [&](int kp, int r) -> uint32_t {
      return (uint32_t)((r / bmsub) * (32 * bmsub * 4) + kp * bmsub * 4 + (r % bmsub) * 4);
    };
    // ---- per-tile state, refreshed when the walk reaches a new tile ----
    // A row r of the tile: sub-block ma = r / 64 of a gang (gang_ma == 2) or
    // row tm*BM + r of the one group; B row r: sub-block nb = r / 64 of a gang
    // (gang_nb > 1) or column tn*BN + r of the one group's B block
    const bool asplit = p.gang_ma == 2, bsplit = p.gang_nb > 1;
    int cur_tile = -1, tm = 0, tn = 0;
    int ga[kGangMA] = {-1, -1}, gb[kGangNB] = {-1, -1, -1, -1};  // groups feeding A / B sub-blocks
    long long b_toff = 0, a_toff = 0;   // element offsets of this thread's first chunk in a block
    uint32_t b_rows_ok = 0;             // bit j: B row br0 + 16 j exists
    bool a_rows_ok = false;             // PLAIN: rows of chunk ach exist
    int a_ma = 0;                       // PLAIN: the A sub-block of chunk ach
    uint32_t v_rows_ok = 0;             // VNNI: bit u: rows of unit u exist
    uint32_t v_ma = 0;                  // VNNI: bit u: unit u reads A sub-block 1
    int v_row[AU];                      // VNNI: first row (within its A block) of unit u
    auto set_tile = [&](int tile) {
      if (p.gang_cells) {
        const int j = tile / p.tiles_n;
        tn = tile - j * p.tiles_n;
        tm = 0;
#pragma unroll
        for (int ma = 0; ma < kGangMA; ++ma) ga[ma] = ma < p.gang_ma ? __ldg(p.gang_rows + j * p.gang_ma + ma) : -1;
#pragma unroll
        for (int nb = 0; nb < kGangNB; ++nb) gb[nb] = nb < p.gang_nb ? __ldg(p.gang_cols + j * p.gang_nb + nb) : -1;
      } else {
        const int per_g = p.tiles_m * p.tiles_n;
        const int g = tile / per_g;
        const int rem = tile - g * per_g;
        tm = rem / p.tiles_n;
        tn = rem - tm * p.tiles_n;
        ga[0] = gb[0] = g;
      }
      b_toff = (long long)((bsplit ? 0 : tn * BN) + br0) * p.ldb + bq * 8;
      b_rows_ok = 0;
#pragma unroll
      for (int jj = 0; jj < BJ; ++jj) {
        const int row = br0 + BRS * jj;
        const int nb = bsplit ? row >> 6 : 0;
        const int rin = bsplit ? (row & 63) : tn * BN + row;
        b_rows_ok |= (uint32_t)(rin < p.n && (nb == 0 ? gb[0] : nb == 1 ? gb[1] : nb == 2 ? gb[2] : gb[3]) >= 0) << jj;
      }
      {
        const int r = ach * 8;
        a_ma = asplit ? r >> 6 : 0;
        const int rin = asplit ? (r & 63) : tm * BM + r;
        a_toff = rin + (long long)akk0 * p.lda;
        a_rows_ok = rin < p.m && (a_ma ? ga[1] : ga[0]) >= 0;
      }
      v_rows_ok = 0;
      v_ma = 0;
#pragma unroll
      for (int u = 0; u < AU; ++u) {
        const int unit = t + u * kProd;
        const int r = (unit % (BM / 4)) * 4;
        const int ma = asplit ? r >> 6 : 0;
        v_row[u] = asplit ? (r & 63) : tm * BM + r;
        v_ma |= (uint32_t)ma << u;
        v_rows_ok |= (uint32_t)(unit < NUNITS && v_row[u] < p.m && (ma ? ga[1] : ga[0]) >= 0) << u;
      }
      cur_tile = tile;
    };
    auto advance = [&](StageIt& s) {
      if (++s.kc == p.kchunks) {
        s.kc = 0;
        if (++s.i == p.count) {
          s.i = 0;
          s.tile += gridDim.x;
        }
      }
    };
    // The batch's index values (STRIDE: the groups' base offsets; OFFSET: the
    // entries' offsets; ADDRESS: their pointers) are staged in shared memory
    // by the producer warps together, kIdxChunk entries at a time (at a tile's
    // first stage and every kIdxChunk entries), one slot per A / B sub-block:
    // a stage then reads them from smem.  A global load per stage whose result
    // the same stage consumes was the producers' critical path -- one L2 round
    // trip per stage, ~0.5 us, with the copies, MMAs and transposes all off.
    const uint32_t sidx = smem_u32(smem + S::IDX_OFF);   // long long [kGangMA + kGangNB][kIdxChunk]
    auto refill = [&](const StageIt& st) {
      named_bar_sync(2, kProd);   // every producer is done with the previous chunk
#pragma unroll
      for (int sl = 0; sl < kGangMA + kGangNB; ++sl) {
        const bool is_a = sl < kGangMA;
        const int g = is_a ? (sl == 0 ? ga[0] : ga[1])
                           : (sl == 2 ? gb[0] : sl == 3 ? gb[1] : sl == 4 ? gb[2] : gb[3]);
        if (g < 0) continue;
        const long long* idx = is_a ? p.a_idx : p.b_idx;
        const uint32_t dst = sidx + sl * kIdxChunk * 8;
        if (p.kind == 0) {
          if (t == 0) sts64(dst, idx ? __ldg(idx + g) : 0);
        } else {
          const long long base = (long long)g * p.count + st.i;
          for (int e = t; e < kIdxChunk && st.i + e < p.count; e += kProd) sts64(dst + e * 8, __ldg(idx + base + e));
        }
      }
      named_bar_sync(2, kProd);
    };
    // per stage: the A / B sub-block base pointers (unused sub-blocks: a valid
    // dummy, their rows are masked)
    const uint16_t* apv[kGangMA];
    const uint16_t* bpv[kGangNB];
    auto stage_ptrs = [&](const StageIt& st) -> bool {
      if ((int)st.tile != cur_tile) set_tile((int)st.tile);
      if (st.kc == 0 && (st.i == 0 || (p.kind != 0 && st.i % kIdxChunk == 0))) refill(st);
      const int e = p.kind == 0 ? 0 : (int)(st.i % kIdxChunk);
      uintptr_t ormask = 0;
      const uint16_t* any = nullptr;   // a real block address: the source of zero-size (masked) copies
      long long vs[kGangMA + kGangNB];  // all index loads first: one smem latency per stage
#pragma unroll
      for (int sl = 0; sl < kGangMA + kGangNB; ++sl) {
        const int g = sl < kGangMA ? (sl == 0 ? ga[0] : ga[1])
                                   : (sl == 2 ? gb[0] : sl == 3 ? gb[1] : sl == 4 ? gb[2] : gb[3]);
        vs[sl] = g >= 0 ? lds64(sidx + (sl * kIdxChunk + e) * 8) : 0;
      }
#pragma unroll
      for (int sl = 0; sl < kGangMA + kGangNB; ++sl) {
        const bool is_a = sl < kGangMA;
        const int g = is_a ? (sl == 0 ? ga[0] : ga[1])
                           : (sl == 2 ? gb[0] : sl == 3 ? gb[1] : sl == 4 ? gb[2] : gb[3]);
        const uint16_t* ptr = nullptr;
        if (g >= 0) {
          const uint16_t* base = is_a ? p.a : p.b;
          const long long v = vs[sl];
          if (p.kind == 0) ptr = base + v + st.i * (is_a ? p.stride_a : p.stride_b);
          else if (p.kind == 1) ptr = base + v;
          else ptr = reinterpret_cast<const uint16_t*>(v);
          ormask |= reinterpret_cast<uintptr_t>(ptr);
          any = ptr;
        }
        if (is_a) apv[sl] = ptr;
        else bpv[sl - kGangMA] = ptr;
      }
#pragma unroll
      for (int ma = 0; ma < kGangMA; ++ma) if (apv[ma] == nullptr) apv[ma] = any;
#pragma unroll
      for (int nb = 0; nb < kGangNB; ++nb) if (bpv[nb] == nullptr) bpv[nb] = any;
      return p.dims_ok && (ormask & 15) == 0;
    };
    // VNNI A fast path: each unit is 4 x 16 B cp.async of words (p, m..m+3)
    // for 4 consecutive k-pairs into this thread's own 64 B of the stage's
    // raw area; once they land (the thread's own cp.async group) the thread
    // word-transposes them into 4 16-byte K-major row chunks of the A tile
    auto issue_vnni = [&](int kc, uint32_t sRaw) {
#pragma unroll
      for (int u = 0; u < AU; ++u) {
        const int unit = t + u * kProd;
        if (unit >= NUNITS) break;
        const int pq = unit / (BM / 4);
        const int k0 = kc * 64 + pq * 8;
        const bool ok = ((v_rows_ok >> u) & 1u) && k0 < p.k;
        const uint16_t* ab = ((v_ma >> u) & 1u) ? apv[1] : apv[0];
        const uint16_t* src = ab + (long long)(k0 >> 1) * 2 * p.m + 2 * v_row[u];
        const uint32_t dst = sRaw + raw_off(pq * 4, (unit % (BM / 4)) * 4);
#pragma unroll
        for (int pp = 0; pp < 4; ++pp)
          cp_async16(dst + pp * bmsub * 4, ok ? (const void*)(src + (long long)pp * 2 * p.m) : (const void*)ab,
                     ok ? 16 : 0);
      }
    };
    auto ld16 = [](const uint16_t* q) -> uint32_t {
      unsigned short v;
      asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(v) : "l"(q));
      return v;
    };
    // fast path: cp.async for B (K-major) and PLAIN A (MN-major)
    auto issue_fast = [&](int kc, uint32_t sA, uint32_t sB) {
      const int kb = kc * 64;
      {
        const bool kok = kb + bq * 8 < p.k;
        const long long step = (long long)BRS * p.ldb;
#pragma unroll
        for (int jj = 0; jj < BJ; ++jj) {
          // split B: rows br0 + 16 jj of sub-block jj / 4 (64 rows each)
          const uint16_t* bb = bsplit ? bpv[(jj >> 2) & 3] : bpv[0];
          const uint16_t* src = bb + b_toff + kb + (bsplit ? (jj & 3) : jj) * step;
          const bool ok = kok && ((b_rows_ok >> jj) & 1u);
          cp_async16(sB + b_soff + jj * BRS * 128, ok ? (const void*)src : (const void*)bb, ok ? 16 : 0);
        }
      }
      if (!p.vnni) {
        const uint16_t* ab = a_ma ? apv[1] : apv[0];
        const uint16_t* src = ab + a_toff + (long long)kb * p.lda;
        const long long step = (long long)AKS * p.lda;
#pragma unroll
        for (int jj = 0; jj < AJ; ++jj) {
          const bool ok = a_rows_ok && kb + akk0 + AKS * jj < p.k;
          cp_async16(sA + a_soff + jj * AKS * 128, ok ? (const void*)(src + jj * step) : (const void*)ab, ok ? 16 : 0);
        }
      }
    };
    // generic path: every chunk from 2-byte loads, bounds per element
    auto issue_generic = [&](int kc, uint32_t sA, uint32_t sB, int tid, int nthr) {
      const int kb = kc * 64;
      for (int c = tid; c < BN * 8; c += nthr) {  // B: column nn, k = kk .. kk+7
        const int r = c >> 3, q = c & 7;
        const int nb = bsplit ? r >> 6 : 0;
        const int nn = bsplit ? (r & 63) : tn * BN + r, kk = kb + q * 8;
        const int g = nb == 0 ? gb[0] : nb == 1 ? gb[1] : nb == 2 ? gb[2] : gb[3];
        const uint16_t* bb = nb == 0 ? bpv[0] : nb == 1 ? bpv[1] : nb == 2 ? bpv[2] : bpv[3];
        uint32_t w[4] = {0, 0, 0, 0};
        if (nn < p.n && g >= 0) {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (kk + e < p.k) w[e >> 1] |= ld16(bb + (long long)nn * p.ldb + kk + e) << (16 * (e & 1));
        }
        sts16(sB + (r >> 3) * 1024 + (r & 7) * 128 + ((q ^ (r & 7)) << 4), make_uint4(w[0], w[1], w[2], w[3]));
      }
      if (!p.vnni) {  // A PLAIN, MN-major chunks: 8 rows at one k
        constexpr int CPR = BM / 8;
        for (int c = tid; c < 64 * CPR; c += nthr) {
          const int kk = c / CPR, ch = c % CPR;
          const int j = ch >> 3, cc = ch & 7;
          const int r = ch * 8, ma = asplit ? r >> 6 : 0;
          const int mrow = asplit ? (r & 63) : tm * BM + r, kg = kb + kk;
          const uint16_t* ab = ma ? apv[1] : apv[0];
          uint32_t w[4] = {0, 0, 0, 0};
          if (kg < p.k && (ma ? ga[1] : ga[0]) >= 0) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (mrow + e < p.m) w[e >> 1] |= ld16(ab + mrow + e + (long long)kg * p.lda) << (16 * (e & 1));
          }
          sts16(sA + j * 8192 + (kk >> 3) * 1024 + (kk & 7) * 128 + ((cc ^ (kk & 7)) << 4),
                make_uint4(w[0], w[1], w[2], w[3]));
        }
      } else {  // A VNNI: the raw unit layout of the fast path (the finisher transposes)
        const uint32_t sRaw = sB + S::B_BYTES;
        for (int unit = tid; unit < NUNITS; unit += nthr) {
          const int pq = unit / (BM / 4), mq = unit % (BM / 4);
          const int r = mq * 4, ma = asplit ? r >> 6 : 0;
          const int r0 = asplit ? (r & 63) : tm * BM + r;
          const uint16_t* ab = ma ? apv[1] : apv[0];
          const bool gok = (ma ? ga[1] : ga[0]) >= 0;
#pragma unroll
          for (int pp = 0; pp < 4; ++pp) {
            const int ke = kb + pq * 8 + 2 * pp;   // k of the pair's even element
            uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
            for (int mm = 0; mm < 4; ++mm) {
              const int mrow = r0 + mm;
              if (gok && mrow < p.m) {
                const uint16_t* q = ab + (long long)(ke >> 1) * 2 * p.m + 2 * mrow;
                if (ke < p.k) w[mm] |= ld16(q);
                if (ke + 1 < p.k) w[mm] |= ld16(q + 1) << 16;
              }
            }
            sts16(sRaw + raw_off(pq * 4 + pp, r), make_uint4(w[0], w[1], w[2], w[3]));
          }
        }
      }
    };
    // issue warps: never wait for data.  A stage's copies arrive on landed[s]
    // as they complete (cp.async.mbarrier.arrive.noinc); the element-wise
    // path writes synchronously, fences and arrives.  Up to STAGES stages in
    // flight, bounded only by the MMA consuming slots.
    StageIt cur{(int)blockIdx.x, 0, 0};
    uint32_t it = 0;
    const bool tr = p.trace && blockIdx.x == 0 && t == 0;
    if (p.tma) {
      // ---- TMA mode: the four producer warps take the stages round-robin
      // (a stage's control code is a serial chain of ~200 instructions; one
      // warp per stage runs four of them at once).  A stage whose blocks do
      // not all start on a row of the maps' views is written element-wise by
      // its warp instead.
      // (at most STAGES warps: a warp's next stage is then never two ring
      // revolutions ahead of the MMA, where the parity wait is ambiguous)
      constexpr int kRR = kProdWarps < STAGES ? kProdWarps : STAGES;
      const int w = warp - kProdWarp0;
      if (lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
      }
      if (w >= kRR) cur.tile = ntiles;
      for (int j = 0; j < w && cur.tile < ntiles; ++j) { advance(cur); ++it; }
      const int asub = p.gang_ma == 2 ? 2 : 1, bsub = bsplit ? p.gang_nb : 1;
      long long abase[kGangMA] = {0, 0}, bbase[kGangNB] = {0, 0, 0, 0};   // STRIDE: the groups' offsets
      const bool trw = p.trace && blockIdx.x == 0 && lane == 0;
      while (cur.tile < ntiles) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        if ((int)cur.tile != cur_tile) {
          set_tile((int)cur.tile);
          if (p.kind == 0) {
#pragma unroll
            for (int ma = 0; ma < kGangMA; ++ma) {
              const int g = ma == 0 ? ga[0] : ga[1];
              abase[ma] = g >= 0 && p.a_idx ? __ldg(p.a_idx + g) : 0;
            }
#pragma unroll
            for (int nb = 0; nb < kGangNB; ++nb) {
              const int g = nb == 0 ? gb[0] : nb == 1 ? gb[1] : nb == 2 ? gb[2] : gb[3];
              bbase[nb] = g >= 0 && p.b_idx ? __ldg(p.b_idx + g) : 0;
            }
          }
        }
        // element offsets of the live blocks (OFFSET: loads issued before
        // the slot wait, used after it)
        long long aoff[kGangMA], boff[kGangNB];
#pragma unroll
        for (int ma = 0; ma < kGangMA; ++ma) {
          const int g = ma == 0 ? ga[0] : ga[1];
          aoff[ma] = g < 0 ? 0
                     : p.kind == 0 ? abase[ma] + cur.i * p.stride_a
                                   : __ldg(p.a_idx + (long long)g * p.count + cur.i);
        }
#pragma unroll
        for (int nb = 0; nb < kGangNB; ++nb) {
          const int g = nb == 0 ? gb[0] : nb == 1 ? gb[1] : nb == 2 ? gb[2] : gb[3];
          boff[nb] = g < 0 ? 0
                     : p.kind == 0 ? bbase[nb] + cur.i * p.stride_b
                                   : __ldg(p.b_idx + (long long)g * p.count + cur.i);
        }
        if (trw && it < kTrace) p.trace[0 * kTrace + it] = clock64();
        mbar_wait(&empty[s], ph ^ 1);
        if (trw && it < kTrace) p.trace[1 * kTrace + it] = clock64();
        long long am = 0, bm = 0;
        const uint16_t* any = nullptr;
#pragma unroll
        for (int ma = 0; ma < kGangMA; ++ma)
          if ((ma == 0 ? ga[0] : ga[1]) >= 0) {
            am |= aoff[ma];
            any = p.a + aoff[ma];
          }
#pragma unroll
        for (int nb = 0; nb < kGangNB; ++nb) bm |= boff[nb];
        // A blocks start on a row of the A view; B blocks on a 64-element
        // chunk of a row of the B view [rows][ldb / 64][64], with the k
        // chunks inside the row
        long long bchunk = 0;
#pragma unroll
        for (int nb = 0; nb < kGangNB; ++nb) bchunk = max(bchunk, ((boff[nb] & ((1LL << p.b_shift) - 1)) >> 6) + p.kchunks);
        const bool rows_ok = ((am & ((1LL << p.a_shift) - 1)) | (bm & 63)) == 0 && bchunk <= (1LL << (p.b_shift - 6)) &&
                             (am >> (p.a_shift + p.a_rbits)) == 0 && (bm >> (p.b_shift + p.b_rbits)) == 0;
        uint8_t* stage = smem + s * S::STAGE;
        if (rows_ok) {
          if (lane == 0) {
            uint32_t bytes = 0;
#pragma unroll
            for (int ma = 0; ma < kGangMA; ++ma)
              if (ma < asub && (ma == 0 ? ga[0] : ga[1]) >= 0) bytes += 128 * bmsub;   // 64 k x bmsub rows
#pragma unroll
            for (int nb = 0; nb < kGangNB; ++nb)
              if (nb < bsub && (nb == 0 ? gb[0] : nb == 1 ? gb[1] : nb == 2 ? gb[2] : gb[3]) >= 0) bytes += 128 * p.b_box;
            mbar_arrive_expect_tx(&landed[s], bytes);
            const int m0 = asplit ? 0 : tm * BM;
#pragma unroll
            for (int ma = 0; ma < kGangMA; ++ma) {
              if (ma >= asub || (ma == 0 ? ga[0] : ga[1]) < 0) continue;
              const int row0 = (int)(aoff[ma] >> p.a_shift);
              if (p.vnni) {   // raw k-pair rows: box {2 bmsub, 32}
                tma_load_5d(stage + S::A_BYTES + S::B_BYTES + ma * 32 * bmsub * 4, &tmA, &landed[s], 2 * m0,
                            row0 + cur.kc * 32, 0, 0, 0);
              } else {        // MN-major 64 x 64 boxes, SW128
                for (int j = 0; j < bmsub / 64; ++j)
                  tma_load_5d(stage + (ma * (bmsub / 64) + j) * 8192, &tmA, &landed[s], m0 + 64 * j,
                              row0 + cur.kc * 64, 0, 0, 0);
              }
            }
#pragma unroll
            for (int nb = 0; nb < kGangNB; ++nb) {
              if (nb >= bsub || (nb == 0 ? gb[0] : nb == 1 ? gb[1] : nb == 2 ? gb[2] : gb[3]) < 0) continue;
              const int row0 = (int)(boff[nb] >> p.b_shift) + (bsplit ? 0 : tn * BN);
              const int ch0 = (int)((boff[nb] & ((1LL << p.b_shift) - 1)) >> 6);
              tma_load_5d(stage + S::A_BYTES + nb * 64 * 128, &tmB, &landed[s], 0, ch0 + cur.kc, row0, 0, 0);
            }
          }
        } else {
          // element-wise by this warp, then its one arrival
#pragma unroll
          for (int ma = 0; ma < kGangMA; ++ma) apv[ma] = (ma == 0 ? ga[0] : ga[1]) >= 0 ? p.a + aoff[ma] : any;
#pragma unroll
          for (int nb = 0; nb < kGangNB; ++nb)
            bpv[nb] = (nb == 0 ? gb[0] : nb == 1 ? gb[1] : nb == 2 ? gb[2] : gb[3]) >= 0 ? p.b + boff[nb] : any;
          const uint32_t sA = smem_u32(stage);
          issue_generic(cur.kc, sA, sA + S::A_BYTES, lane, 32);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&landed[s]);
        }
        if (trw && it < kTrace) p.trace[2 * kTrace + it] = clock64();
        for (int j = 0; j < kRR && cur.tile < ntiles; ++j) { advance(cur); ++it; }
      }
    }
    while (!p.tma && cur.tile < ntiles) {
      const int s = it % STAGES;
      const uint32_t ph = (it / STAGES) & 1;
      const bool fast = stage_ptrs(cur);
      if (tr && it < kTrace) p.trace[0 * kTrace + it] = clock64();
      if (p.dbg & 8) mbar_wait_sleep(&empty[s], ph ^ 1); else mbar_wait(&empty[s], ph ^ 1);
      if (tr && it < kTrace) p.trace[1 * kTrace + it] = clock64();
      const uint32_t sA = smem_u32(smem + s * S::STAGE), sB = sA + S::A_BYTES;
      if (p.dbg & 2) {
        mbar_arrive(&landed[s]);
      } else if (fast) {
        issue_fast(cur.kc, sA, sB);
        if (p.vnni) issue_vnni(cur.kc, sB + S::B_BYTES);
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&landed[s])) : "memory");
      } else {
        issue_generic(cur.kc, sA, sB, t, kProd);
        fence_async_smem();
        mbar_arrive(&landed[s]);
      }
      if (tr && it < kTrace) p.trace[2 * kTrace + it] = clock64();
      advance(cur);
      ++it;
    }
  } else if (warp >= kFinWarp0 && warp < kFinWarp0 + kFinWarps) {
    // ============================ finishers ============================
    // per landed stage: VNNI A's word transpose (raw -> K-major A tile), then
    // the generic -> async proxy fence the tensor core's operand reads need,
    // then full[s] for the MMA warp
    const int t = threadIdx.x - kFinWarp0 * 32;
    const int bmsub = p.gang_ma == 2 ? 64 : BM;
    constexpr int AU = (BM * 2 + 32 * kFinWarps - 1) / (32 * kFinWarps);
    constexpr int NUNITS = BM * 2;
    const int per_tile = (int)(p.count * p.kchunks);
    const int my_tiles = ntiles > (int)blockIdx.x ? (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    const long long nst = (long long)my_tiles * per_tile;
    for (long long it = 0; it < nst; ++it) {
      const int s = (int)(it % STAGES);
      if (p.dbg & 8) mbar_wait_sleep(&landed[s], (uint32_t)((it / STAGES) & 1)); else mbar_wait(&landed[s], (uint32_t)((it / STAGES) & 1));
      if (p.trace && blockIdx.x == 0 && t == 0 && it < kTrace) p.trace[3 * kTrace + it] = clock64();
      if (TA) {
        // row q*32 + lane of the A tile: its 32 k-pair words -> TMEM columns
        // 2 BN + 32 s .. (lane quarter q = warp % 4)
        tc_fence_after();
        const int q = warp & 3, r = q * 32 + lane;
        const uint32_t sRaw = smem_u32(smem + s * S::STAGE) + S::A_BYTES + S::B_BYTES +
                              (uint32_t)((r / bmsub) * (32 * bmsub * 4) + (r % bmsub) * 4);
        uint32_t w[32];
#pragma unroll
        for (int kp = 0; kp < 32; ++kp)
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[kp]) : "r"(sRaw + kp * bmsub * 4));
        tmem_st32(tmem_base + ((uint32_t)(q * 32) << 16) + 2 * BN + s * 32, w);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
        if (p.trace && blockIdx.x == 0 && t == 0 && it < kTrace) p.trace[4 * kTrace + it] = clock64();
        continue;
      }
      if (p.vnni && !(p.dbg & 4)) {
        const uint32_t sA = smem_u32(smem + s * S::STAGE), sRaw = sA + S::A_BYTES + S::B_BYTES;
#pragma unroll
        for (int u = 0; u < AU; ++u) {
          const int unit = t + u * 32 * kFinWarps;
          if (unit >= NUNITS) break;
          const int pq = unit / (BM / 4), mq = unit % (BM / 4);
          // raw [sub-block][k-pair][row] words: consecutive lanes read
          // consecutive 16 B (no bank conflicts)
          const int r0 = mq * 4;
          const uint32_t src = sRaw + (uint32_t)((r0 / bmsub) * (32 * bmsub * 4) + pq * 4 * bmsub * 4 + (r0 % bmsub) * 4);
          uint4 r[4];
#pragma unroll
          for (int pp = 0; pp < 4; ++pp)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(r[pp].x), "=r"(r[pp].y), "=r"(r[pp].z), "=r"(r[pp].w)
                         : "r"(src + pp * bmsub * 4));
          // write j: row mq*4 + (j + rot) & 3, rotated by lane so that any 8
          // consecutive lanes hit 8 different 16-byte bank groups (the same
          // row offset for all lanes puts a warp's 32 chunks on 2 of them);
          // the words are rotated once with predicated selects (no branches)
          const int rot = (lane >> 1) & 3;
#pragma unroll
          for (int pp = 0; pp < 4; ++pp) r[pp] = rot4(r[pp], rot);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int row = mq * 4 + ((j + rot) & 3);
            const uint32_t w0 = j == 0 ? r[0].x : j == 1 ? r[0].y : j == 2 ? r[0].z : r[0].w;
            const uint32_t w1 = j == 0 ? r[1].x : j == 1 ? r[1].y : j == 2 ? r[1].z : r[1].w;
            const uint32_t w2 = j == 0 ? r[2].x : j == 1 ? r[2].y : j == 2 ? r[2].z : r[2].w;
            const uint32_t w3 = j == 0 ? r[3].x : j == 1 ? r[3].y : j == 2 ? r[3].z : r[3].w;
            sts16(sA + (row >> 3) * 1024 + (row & 7) * 128 + ((pq ^ (row & 7)) << 4), make_uint4(w0, w1, w2, w3));
          }
        }
      }
      // every thread orders its own transposed chunks for the async proxy, then
      // one elected arrival per warp (128 arrivals on one mbarrier word per
      // stage serialise in shared memory)
      if (!(p.dbg & 32)) fence_async_smem();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&full[s]);
      if (p.trace && blockIdx.x == 0 && t == 0 && it < kTrace) p.trace[4 * kTrace + it] = clock64();
    }
  } else if (warp == kMmaWarp) {
    // ============================ MMA issue ============================
    const uint32_t idesc = idesc_bf16_f32(BM, BN, p.vnni ? 0 : 1, 0);
    const uint64_t a0 = p.vnni ? sw128_kmajor_desc(smem_u32(smem)) : sw128_mnmajor_desc(smem_u32(smem), 8192);
    const uint64_t b0 = sw128_kmajor_desc(smem_u32(smem + S::A_BYTES));
    const uint32_t astep = p.vnni ? (32 >> 4) : (2048 >> 4);
    uint32_t it = 0, tcount = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tcount) {
      const uint32_t as = tcount & 1, aph = (tcount >> 1) & 1;
      mbar_wait(&tempty[as], aph ^ 1);
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + as * BN;
      for (long long j = 0; j < per_tile; ++j, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        if (p.trace && blockIdx.x == 0 && lane == 0 && it < kTrace) p.trace[5 * kTrace + it] = clock64();
        tc_fence_after();
        const uint64_t soff = (uint64_t)((s * S::STAGE) >> 4);
        if (TA) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_f16_tmem_a_warp(tmem_d, tmem_base + 2 * BN + s * 32 + kk * 8, b0 + soff + 2 * kk, idesc,
                                 (j > 0 || kk > 0) ? 1u : 0u);
        } else {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            if (!(p.dbg & 1))
              umma_f16_warp(tmem_d, a0 + soff + astep * kk, b0 + soff + 2 * kk, idesc, (j > 0 || kk > 0) ? 1u : 0u);
        }
        if (p.dbg & 16) {
          if (lane == 0) mbar_arrive(&empty[s]);
        } else {
          umma_commit_warp(&empty[s]);
        }
      }
      umma_commit_warp(&tfull[as]);
    }
  } else if (warp < kEpiWarps) {
    // ============================ epilogue ============================
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int q = warp;
    // accumulator row of this lane: M = 128 -> lane q*32 + l; M = 64 -> the
    // 64 rows sit in lanes 0-15 of each 32-lane quarter
    const int lrow = BM == 128 ? q * 32 + lane : q * 16 + lane;
    const bool lane_ok = BM == 128 || lane < 16;
    uint32_t tcount = 0;
    const bool asplit = p.gang_ma == 2, bsplit = p.gang_nb > 1;
    const int ma = asplit ? lrow >> 6 : 0;   // this lane's A sub-block (gangs)
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tcount) {
      int tm, tn, row;
      // C blocks of this lane's row: one per B sub-block (gangs) or the group's
      float* cgs[kGangNB] = {nullptr, nullptr, nullptr, nullptr};
      // (BF16 output: the same pointers carry uint16_t element offsets)
      auto cptr = [&](long long off) -> float* {
        return p.c16 ? reinterpret_cast<float*>(p.c16 + off) : p.c + off;
      };
      if (p.gang_cells) {
        const int j = tile / p.tiles_n;
        tn = tile - j * p.tiles_n;
        tm = 0;
        row = asplit ? (lrow & 63) : lrow;
#pragma unroll
        for (int nb = 0; nb < kGangNB; ++nb) {
          const int cell = nb < p.gang_nb && ma < p.gang_ma ? __ldg(p.gang_cells + (j * p.gang_ma + ma) * p.gang_nb + nb)
                                                            : -1;
          cgs[nb] = cell >= 0 ? cptr(p.c_off ? p.c_off[cell] : 0) : nullptr;
        }
      } else {
        const int per_g = p.tiles_m * p.tiles_n;
        const int g = tile / per_g;
        const int rem = tile - g * per_g;
        tm = rem / p.tiles_n;
        tn = rem - tm * p.tiles_n;
        row = tm * BM + lrow;
        cgs[0] = cptr(p.c_off ? p.c_off[g] : 0);
      }
      const bool row_ok = lane_ok && row < p.m;
      const uint32_t as = tcount & 1, aph = (tcount >> 1) & 1;
      if (p.dbg & 8) mbar_wait_sleep(&tfull[as], aph); else mbar_wait(&tfull[as], aph);
      if (p.trace && blockIdx.x == 0 && threadIdx.x == 0 && tcount < 8) p.trace[6 * kTrace + 2 * tcount] = clock64();
      tc_fence_after();
      const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + as * BN;
      uint32_t v[32];
#pragma unroll 1
      for (int ch = 0; ch < BN / 32; ++ch) {
        tmem_ld32(tacc + ch * 32, v);
        tmem_ld_wait();
        if (p.trace && blockIdx.x == 0 && threadIdx.x == 0 && tcount == 0 && ch < 8) p.trace[6 * kTrace + 32 + ch] = clock64();
        if (ch == BN / 32 - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[as]);
        }
        // split B: chunk ch is columns (ch & 1) * 32 .. of B sub-block ch / 2
        const int nbc = bsplit ? ch >> 1 : 0;
        float* cg = nbc == 0 ? cgs[0] : nbc == 1 ? cgs[1] : nbc == 2 ? cgs[2] : cgs[3];
        const int col0 = bsplit ? (ch & 1) * 32 : tn * BN + ch * 32;
        if (p.c16) {
          if (row_ok && cg != nullptr) {
            // straight-line: per column a multiply-high division and a
            // predicated 2-byte store (a branch per column serialised them)
            uint16_t* cb = reinterpret_cast<uint16_t*>(cg) + row;
            const unsigned per = (unsigned)p.col_period, keep = (unsigned)p.col_keep, nn = (unsigned)p.n;
            const unsigned r0 = __umulhi((unsigned)col0, p.col_magic), c0 = (unsigned)col0 - r0 * per;
            if (c0 + 32 <= keep && (unsigned)col0 + 32 <= nn) {
              // the chunk inside one kept row segment: columns map linearly
              uint16_t* dst = cb + (long long)(r0 * keep + c0) * p.ldc;
              const long long ld = p.ldc;
#pragma unroll
              for (int i = 0; i < 32; ++i) dst[i * ld] = f32_to_bf16(__uint_as_float(v[i]));
            } else
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const unsigned vc = (unsigned)col0 + i;
              const unsigned orow = __umulhi(vc, p.col_magic);
              const unsigned ocol = vc - orow * per;
              const int ok = vc < nn && ocol < keep;
              uint16_t* dst = cb + (long long)(orow * keep + ocol) * p.ldc;
              const uint16_t hv = f32_to_bf16(__uint_as_float(v[i]));
              asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %2, 0;\n\t@q st.global.u16 [%0], %1;\n\t}"
                           ::"l"(dst), "h"(hv), "r"(ok) : "memory");
            }
          }
        } else if (row_ok && cg != nullptr && p.beta_mode == 0 && col0 + 32 <= p.n) {
          // whole chunk, beta = 0: 32 independent stores (one basic block;
          // a per-store beta / bounds branch serialised them, ~45 cycles each)
          float* dst = cg + row + (long long)col0 * p.ldc;
          const long long ld = p.ldc;
#pragma unroll
          for (int i = 0; i < 32; ++i) dst[i * ld] = __uint_as_float(v[i]);
        } else if (row_ok && cg != nullptr) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int col = col0 + i;
            if (col < p.n) {
              float* dst = cg + row + (long long)col * p.ldc;
              const float acc = __uint_as_float(v[i]);
              *dst = p.beta_mode == 0 ? acc : p.beta_mode == 1 ? __fadd_rn(*dst, acc)
                                                               : __fadd_rn(__fmul_rn(*dst, p.beta), acc);
            }
          }
        }
      }
      if (p.trace && blockIdx.x == 0 && threadIdx.x == 0 && tcount < 8) p.trace[6 * kTrace + 2 * tcount + 1] = clock64();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem_base, tcols);
  }
}

template <int BM, int BN, int STAGES, bool TA = false>
static int launch(GParams p, cudaStream_t s) {
  using S = GSmem<BM, BN, STAGES, TA>;
  static_assert(!TA || (BM == 128 && 2 * BN + STAGES * 32 <= 512), "TMEM: accumulators + A stages");
  p.tmem_a = TA;
  CUtensorMap ma, mb;
  memset(&ma, 0, sizeof(ma));
  memset(&mb, 0, sizeof(mb));
  if (p.tma) {
    const int bmsub = p.gang_ma == 2 ? 64 : BM;
    // row counts: 2^30 at most, and the outer strides (rows x pitch) < 2^39 B
    auto rbits = [](uint64_t pitch) { int b = kTmaRowBits; while (b > 0 && (pitch << b) >= (1ull << 39)) --b; return b; };
    const uint64_t pa = (uint64_t)(p.vnni ? 4 * p.m : 2 * p.lda), pb = (uint64_t)(2 * p.ldb);
    p.a_rbits = rbits(pa);
    p.b_rbits = rbits(pb);
    const uint64_t R = 1ull << p.a_rbits;
    uint64_t da[5] = {(uint64_t)(p.vnni ? 2 * p.m : p.m), R, 1, 1, 1};
    uint64_t sa[4] = {pa, 0, 0, 0};
    uint32_t ba[5] = {(uint32_t)(p.vnni ? 2 * bmsub : 64), (uint32_t)(p.vnni ? 32 : 64), 1, 1, 1};
    sa[1] = sa[0] * R; sa[2] = sa[1]; sa[3] = sa[1];
    int rc = make_tma_map_5d(&ma, p.a, da, sa, ba, p.vnni ? 0 : 128);
    // B view [rows][ldb / 64][64]: a block may start on any 64-element chunk
    const uint64_t RB = 1ull << p.b_rbits;
    uint64_t db[5] = {64, (uint64_t)(p.ldb / 64), RB, 1, 1};
    uint64_t sb[4] = {128, pb, 0, 0};
    sb[2] = sb[1] * RB; sb[3] = sb[2];
    uint32_t bb[5] = {64, 1, (uint32_t)p.b_box, 1, 1};
    if (rc == TPP_OK) rc = make_tma_map_5d(&mb, p.b, db, sb, bb, 128);
    if (rc != TPP_OK) p.tma = 0;   // (a map the driver rejects: the cp.async path)
  }
  static_assert(S::BYTES <= 227 * 1024, "shared memory budget");
  auto kern = brgemm_grouped_kernel<BM, BN, STAGES, TA>;
  cudaError_t e = ensure_smem_attr((const void*)kern, S::BYTES);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(brgemm_grouped_kernel)");
  const long long ntiles = p.gang_cells ? (long long)p.ngangs * p.tiles_n : p.groups * p.tiles_m * p.tiles_n;
  const int grid = (int)(ntiles < num_sms() ? ntiles : num_sms());
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = S::BYTES;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_allowed();
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, ma, mb, p);
  if (e != cudaSuccess) return cuda_status(e, "cudaLaunchKernelEx(brgemm_grouped_kernel)");
  TPP_CUDA_LAUNCH_CHECK("brgemm_grouped_kernel");
  if (p.trace) {   // probe: dump CTA 0's stamps (cycles from kernel entry)
    long long h[8 * kTrace];
    cudaStreamSynchronize(s);
    cudaMemcpy(h, p.trace, sizeof(h), cudaMemcpyDeviceToHost);
    const long long t0 = h[7 * kTrace];
    fprintf(stderr, "grp trace <%d,%d,%d>: it  prod_ready empty_ok issued | landed full_arr | mma_full\n", BM, BN, STAGES);
    for (int i = 0; i < kTrace; ++i) {
      if (h[5 * kTrace + i] == 0) break;
      fprintf(stderr, "  %3d %7lld %7lld %7lld | %7lld %7lld | %7lld\n", i, h[i] - t0, h[kTrace + i] - t0,
              h[2 * kTrace + i] - t0, h[3 * kTrace + i] - t0, h[4 * kTrace + i] - t0, h[5 * kTrace + i] - t0);
    }
    for (int c = 0; c < 8 && h[6 * kTrace + 32 + c]; ++c) fprintf(stderr, "  tile 0 chunk %d loaded %lld\n", c, h[6 * kTrace + 32 + c] - t0);
    for (int j = 0; j < 8 && h[6 * kTrace + 2 * j]; ++j)
      fprintf(stderr, "  tile %d: tfull %lld epi_done %lld\n", j, h[6 * kTrace + 2 * j] - t0, h[6 * kTrace + 2 * j + 1] - t0);
  }
  set_last_config("brgemm_grouped_kernel<" + std::to_string(BM) + "," + std::to_string(BN) + "," +
                  std::to_string(STAGES) + "> grid=" + std::to_string(grid) + " tiles=" + std::to_string(ntiles) +
                  (p.gang_cells ? " gang=" + std::to_string(p.gang_ma) + "x" + std::to_string(p.gang_nb) : "") +
                  (p.tma ? " tma" : "") + (p.tmem_a ? " tmem_a" : ""));
  return TPP_OK;
}

}  // namespace grp

// 1 = not applicable (caller falls back to the ordered engine), else a status
int brgemm_grouped_tc(const tpp_gemm_desc* d, int kind, const void* a, const void* b, int64_t stride_a,
                      int64_t stride_b, const int64_t* a_idx, const int64_t* b_idx, int64_t count, void* c,
                      const int64_t* c_off, int64_t groups, cudaStream_t s, const int32_t* gang, int ngangs,
                      int gang_ma, int gang_nb, void* c_bf16, int col_period, int col_keep) {
  using namespace grp;
  if (d->in_dtype != TPP_BF16 || count < 1 || groups < 1) return 1;
  GParams p{};
  p.gang_ma = 1;
  p.gang_nb = 1;
  if (gang != nullptr) {
    TPP_REQUIRE(ngangs >= 1 && (gang_ma == 1 || gang_ma == 2) && (gang_nb == 1 || gang_nb == 2 || gang_nb == 4),
                TPP_E_TENSOR, "gangs: 1 or 2 A sub-blocks x 1, 2 or 4 B sub-blocks");
    TPP_REQUIRE(d->m <= 64 && (gang_nb == 1 || d->n <= 64), TPP_E_UNSUPPORTED,
                "gangs stack 64-row A blocks (m <= 64) and, for several B sub-blocks, 64-column B blocks (n <= 64)");
    p.gang_ma = gang_ma;
    p.gang_nb = gang_nb;
    p.ngangs = ngangs;
    p.gang_rows = gang;
    p.gang_cols = gang + (int64_t)ngangs * gang_ma;
    p.gang_cells = gang + (int64_t)ngangs * (gang_ma + gang_nb);
  }
  // fast-path shape condition; block alignment is checked per stage in the kernel
  p.dims_ok = !(d->k % 8 || d->m % 8 || d->ldb % 8 || (!d->a_vnni && d->lda % 8));
  p.m = d->m; p.n = d->n; p.k = d->k;
  p.lda = d->lda; p.ldb = d->ldb; p.ldc = d->ldc;
  p.vnni = d->a_vnni;
  p.kind = kind;
  p.a = reinterpret_cast<const uint16_t*>(a);
  p.b = reinterpret_cast<const uint16_t*>(b);
  p.stride_a = stride_a; p.stride_b = stride_b;
  p.a_idx = reinterpret_cast<const long long*>(a_idx);
  p.b_idx = reinterpret_cast<const long long*>(b_idx);
  p.count = count;
  p.c = reinterpret_cast<float*>(c);
  p.c16 = reinterpret_cast<uint16_t*>(c_bf16);
  p.col_period = col_period > 0 ? col_period : d->n;
  p.col_keep = col_keep > 0 ? col_keep : p.col_period;
  p.col_magic = (unsigned)((0x100000000ull + (unsigned long long)p.col_period - 1) / (unsigned long long)p.col_period);
  TPP_REQUIRE(!c_bf16 || (long long)d->n * p.col_period < (1LL << 31), TPP_E_UNSUPPORTED,
              "BF16 output column map: n x col_period < 2^31");
  TPP_REQUIRE(!c_bf16 || d->beta == 0.0, TPP_E_TENSOR, "BF16 output needs beta = 0");
  p.c_off = reinterpret_cast<const long long*>(c_off);
  p.groups = groups;
  p.kchunks = (d->k + 63) / 64;
  p.beta = (float)d->beta;
  p.beta_mode = d->beta == 0.0 ? 0 : d->beta == 1.0 ? 1 : 2;
  static const int dbg = getenv("TPP_GRP_DBG") ? atoi(getenv("TPP_GRP_DBG")) : 0;
  p.dbg = dbg;
  if (getenv("TPP_GRP_TRACE")) {
    static long long* tbuf = nullptr;
    if (!tbuf) cudaMalloc(&tbuf, 8 * kTrace * sizeof(long long));
    cudaMemsetAsync(tbuf, 0, 8 * kTrace * sizeof(long long), s);
    p.trace = tbuf;
  }
  const int BM = gang ? 64 * gang_ma : (d->m <= 64 ? 64 : 128);
  // widest N tile that still gives every SM a tile (one C block of a
  // single brgemm() call is otherwise only a handful of work items)
  const long long tm_all = gang ? ngangs : groups * ((d->m + BM - 1) / BM);
  int BN = d->n <= 64 ? 64 : d->n <= 128 ? 128 : 256;
  while (BN > 64 && tm_all * ((d->n + BN - 1) / BN) < num_sms()) BN /= 2;
  if (gang && gang_nb > 1) BN = 64 * gang_nb;
  p.tiles_m = gang ? 1 : (d->m + BM - 1) / BM;
  p.tiles_n = gang && gang_nb > 1 ? 1 : (d->n + BN - 1) / BN;
  TPP_REQUIRE(tm_all * p.tiles_m * p.tiles_n < (1LL << 31), TPP_E_UNSUPPORTED, "grouped BRGEMM: too many tiles");
  {
    // TMA staging: power-of-two row pitches (a block's first row is then a
    // shift of its offset, checked per stage), whole 64-k chunks, B tiles
    // that are whole boxes; ADDRESS batches keep the cp.async path
    static const bool no_tma = getenv("TPP_GRP_NO_TMA") != nullptr;
    auto pow2 = [](long long v) { return v > 0 && (v & (v - 1)) == 0; };
    auto lg2 = [](long long v) { int r = 0; while ((1LL << r) < v) ++r; return r; };
    const long long pa = d->a_vnni ? 2LL * d->m : d->lda;
    const int bn_sub = gang && gang_nb > 1 ? 64 : BN;
    const int b_box = d->n < bn_sub ? d->n : bn_sub;
    const bool ok = !no_tma && kind != 2 && d->k % 64 == 0 && pow2(pa) && pa >= 8 && pow2(d->ldb) && d->ldb >= 64 &&
                    d->n % 8 == 0 && d->n % b_box == 0 && reinterpret_cast<uintptr_t>(a) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(b) % 16 == 0;
    p.tma = ok ? 1 : 0;
    p.a_shift = lg2(pa);
    p.b_shift = lg2(d->ldb);
    p.b_box = b_box;
  }
  if (BM == 64) {
    if (BN == 64) return launch<64, 64, 8>(p, s);
    if (BN == 128) return launch<64, 128, 6>(p, s);
    return launch<64, 256, 4>(p, s);
  }
  static const bool no_tmem_a = getenv("TPP_GRP_NO_TMEM_A") != nullptr;
  if (p.vnni && BN <= 128 && !no_tmem_a) {   // VNNI A through tensor memory, deeper rings
    if (BN == 64) return launch<128, 64, 8, true>(p, s);
    return launch<128, 128, 6, true>(p, s);
  }
  if (BN == 64) return launch<128, 64, 5>(p, s);
  if (BN == 128) return launch<128, 128, 4>(p, s);
  return launch<128, 256, 3>(p, s);
}

}  // namespace tpp

// K6: layout transforms (bit-exact, HBM-bound).
//
//  * weight packing VNNI -> UMMA-canonical K-major blocks.  A VNNI-2 block
//    [K/2][M][2] (contraction.py:238-247) viewed as 32-bit words is a
//    (K/2) x M word matrix; its word transpose is [M][K] K-major, the layout
//    the tcgen05 B operand (and TMA 128B swizzle) wants.  Done once per
//    weight tensor (inference) or once per step (training).
//  * the transform TPP (ops.py:537-570): TRANSPOSE, VNNI, VNNI_TO_VNNIT on
//    column-major views.

#include "common.cuh"

namespace tpp {

// ---- word transpose of many (rows x cols) 32-bit blocks, with block remap ----
// src block b (contiguous rows*cols words) -> dst block remap(b), transposed.
__device__ __forceinline__ int64_t remap_block(const BlockRemap& r, int64_t b) {
  if (r.mode == 0) return b;
  const int i3 = (int)(b % r.d3);
  int64_t t = b / r.d3;
  const int i2 = (int)(t % r.d2);
  t /= r.d2;
  const int i1 = (int)(t % r.d1);
  const int i0 = (int)(t / r.d1);
  // conv fwd: src [Kb][Cb][R][S] -> dst [Kb][R][S][Cb]
  return (((int64_t)i0 * r.d2 + i2) * r.d3 + i3) * r.d1 + i1;
}

__global__ void word_transpose_blocks(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                      int rows, int cols, BlockRemap remap) {
  __shared__ uint32_t tile[32][33];
  const int64_t b = blockIdx.z;
  const uint32_t* s = src + b * (int64_t)rows * cols;
  uint32_t* d = dst + remap_block(remap, b) * (int64_t)rows * cols;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = s[(int64_t)r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) d[(int64_t)c * rows + r] = tile[threadIdx.x][i];
  }
}

int launch_word_transpose_blocks(const void* src, void* dst, int rows, int cols, int64_t nblocks,
                                 BlockRemap remap, cudaStream_t s) {
  if (nblocks == 0) return TPP_OK;
  TPP_REQUIRE(nblocks < 65536, TPP_E_UNSUPPORTED, "too many weight blocks for one pack launch");
  dim3 grid((cols + 31) / 32, (rows + 31) / 32, (unsigned)nblocks);
  word_transpose_blocks<<<grid, dim3(32, 8), 0, s>>>(reinterpret_cast<const uint32_t*>(src),
                                                      reinterpret_cast<uint32_t*>(dst), rows, cols,
                                                      remap);
  TPP_CUDA_LAUNCH_CHECK("word_transpose_blocks");
  return TPP_OK;
}

// conv backward-data weights: VNNI [Kb][Cb][R][S][bc/2][bk][2] ->
// [Cb][R][S][Kb][bc][bk] with taps flipped (out channel c, reduce over k):
// dst[cb][R-1-r][S-1-s][kb][c][k] = src[kb][cb][r][s][c/2][k][c%2]
__global__ void pack_conv_bwd_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst,
                                     int Kb, int Cb, int R, int S, int bc, int bk) {
  const int64_t total = (int64_t)Kb * Cb * R * S * bc * bk;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e % bk);
    int64_t t = e / bk;
    const int c = (int)(t % bc);
    t /= bc;
    const int kb = (int)(t % Kb);
    t /= Kb;
    const int sf = (int)(t % S);
    t /= S;
    const int rf = (int)(t % R);
    const int cb = (int)(t / R);
    const int r = R - 1 - rf, s = S - 1 - sf;
    const int64_t blk = (((int64_t)kb * Cb + cb) * R + r) * S + s;
    dst[e] = src[blk * bc * bk + (int64_t)(c >> 1) * bk * 2 + k * 2 + (c & 1)];
  }
}

int launch_pack_conv_bwd(const void* src, void* dst, int Kb, int Cb, int R, int S, int bc, int bk,
                         cudaStream_t s) {
  const int64_t total = (int64_t)Kb * Cb * R * S * bc * bk;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 65536) blocks = 65536;
  pack_conv_bwd_kernel<<<(unsigned)blocks, threads, 0, s>>>(
      reinterpret_cast<const uint16_t*>(src), reinterpret_cast<uint16_t*>(dst), Kb, Cb, R, S, bc, bk);
  TPP_CUDA_LAUNCH_CHECK("pack_conv_bwd_kernel");
  return TPP_OK;
}

// Backward-data weights in the reference VNNI layout (the generic conv path
// runs them as offset-BRGEMM A blocks): block (cb, kb, r', s') =
// VNNI_TO_VNNIT of forward block (kb, cb, R-1-r', S-1-s') -- logical (c x k),
// stored [k/2][c][2] (ops.py:556-565 on a spatial flip; the oracle's
// conv_weights_bwd_data).
__global__ void pack_conv_bwd_vnni_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst,
                                          int Kb, int Cb, int R, int S, int bc, int bk) {
  const int64_t total = (int64_t)Kb * Cb * R * S * bc * bk;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int pb = (int)(e & 1);
    int64_t t = e >> 1;
    const int c = (int)(t % bc);
    t /= bc;
    const int k = 2 * (int)(t % (bk / 2)) + pb;
    t /= bk / 2;
    const int sf = (int)(t % S);
    t /= S;
    const int rf = (int)(t % R);
    t /= R;
    const int kb = (int)(t % Kb);
    const int cb = (int)(t / Kb);
    const int64_t blk = (((int64_t)kb * Cb + cb) * R + (R - 1 - rf)) * S + (S - 1 - sf);
    dst[e] = src[blk * bc * bk + (int64_t)(c >> 1) * bk * 2 + k * 2 + (c & 1)];
  }
}

int launch_pack_conv_bwd_vnni(const void* src, void* dst, int Kb, int Cb, int R, int S, int bc, int bk,
                              cudaStream_t s) {
  const int64_t total = (int64_t)Kb * Cb * R * S * bc * bk;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 65536) blocks = 65536;
  pack_conv_bwd_vnni_kernel<<<(unsigned)blocks, threads, 0, s>>>(
      reinterpret_cast<const uint16_t*>(src), reinterpret_cast<uint16_t*>(dst), Kb, Cb, R, S, bc, bk);
  TPP_CUDA_LAUNCH_CHECK("pack_conv_bwd_vnni_kernel");
  return TPP_OK;
}

// Explicit zero padding (and zero insertion) of a blocked activation
// [N][C_b][Hi][Wi][64] into [N][C_b][Ho][Wo][64]: output pixel (y, x) is input
// ((y - top) / dil, (x - left) / dil) when both divide evenly and land inside
// the input, else 0 -- the padded input the reference's offset-BRGEMM
// convolution reads (dil > 1: the zero-inserted dO of a strided conv's
// backward-data).  16 bytes (8 channels) per thread.
__global__ void conv_pad_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, int64_t planes, int hi,
                                int wi, int ho, int wo, int top, int left, int dil) {
  const int64_t total = planes * ho * wo * 8;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(e & 7);
    int64_t t = e >> 3;
    const int x = (int)(t % wo);
    t /= wo;
    const int y = (int)(t % ho);
    const int64_t pl = t / ho;
    const int yy = y - top, xx = x - left;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (yy >= 0 && xx >= 0 && yy % dil == 0 && xx % dil == 0 && yy / dil < hi && xx / dil < wi)
      v = in[((pl * hi + yy / dil) * wi + xx / dil) * 8 + q];
    out[e] = v;
  }
}

int launch_conv_pad(const void* in, void* out, int64_t planes, int hi, int wi, int ho, int wo, int top, int left,
                    int dil, cudaStream_t s) {
  const int64_t total = planes * ho * wo * 8;
  if (total == 0) return TPP_OK;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  conv_pad_kernel<<<(unsigned)blocks, threads, 0, s>>>(reinterpret_cast<const uint4*>(in), reinterpret_cast<uint4*>(out),
                                                       planes, hi, wi, ho, wo, top, left, dil);
  TPP_CUDA_LAUNCH_CHECK("conv_pad_kernel");
  return TPP_OK;
}

// ---- transform TPP (ops.py:537-570) on column-major views -----------------
// Elements are moved as raw bits of `esize` bytes.
template <typename T>
__global__ void transform_kernel(int kind, const T* __restrict__ in, int in_ld, T* __restrict__ out,
                                 int out_rows, int out_cols, int out_ld, int alpha, int alpha_out,
                                 int lrows, int lcols) {
  const int64_t total = (int64_t)out_rows * out_cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % out_rows);  // output physical row
    const int j = (int)(e / out_rows);  // output physical col
    T v = T(0);
    if (kind == 0) {
      // TRANSPOSE: out(i, j) = in(j, i)
      v = in[j + (int64_t)i * in_ld];
    } else if (kind == 1) {
      // VNNI: out flat [g][m][r] = L(m, g*alpha + r); out phys (m*alpha + r, g)
      const int m = i / alpha, r = i % alpha;
      const int src_col = j * alpha + r;
      if (src_col < lcols) v = in[m + (int64_t)src_col * in_ld];
    } else if (kind == 3) {
      v = in[i + (int64_t)j * in_ld];  // COPY
    } else {
      // VNNI_TO_VNNIT: out = vnni_pack(L^T, alpha_out), L = vnni_unpack(in, alpha, lrows, lcols)
      // out phys (m*alpha_out + r, g): L^T(m, g*alpha_out + r) = L(g*alpha_out + r, m)
      const int m = i / alpha_out, r = i % alpha_out;
      const int li = j * alpha_out + r, lj = m;
      if (li < lrows) v = in[(int64_t)(li * alpha + lj % alpha) + (int64_t)(lj / alpha) * in_ld];
    }
    out[i + (int64_t)j * out_ld] = v;
  }
}

int launch_transform(int kind, int esize, const void* in, int in_ld, void* out, int out_rows,
                     int out_cols, int out_ld, int alpha, int alpha_out, int lrows, int lcols,
                     cudaStream_t s) {
  const int64_t total = (int64_t)out_rows * out_cols;
  if (total == 0) return TPP_OK;
  if (kind <= 2) {
    const int rc = fast_transform(kind, esize, in, in_ld, out, out_rows, out_cols, out_ld, alpha, alpha_out, lrows,
                                  lcols, s);
    if (rc == 0) return TPP_OK;
    if (rc == 2) return cuda_status(cudaGetLastError(), "fast transform");
  }
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 65536) blocks = 65536;
  switch (esize) {
    case 1:
      transform_kernel<uint8_t><<<(unsigned)blocks, threads, 0, s>>>(
          kind, (const uint8_t*)in, in_ld, (uint8_t*)out, out_rows, out_cols, out_ld, alpha,
          alpha_out, lrows, lcols);
      break;
    case 2:
      transform_kernel<uint16_t><<<(unsigned)blocks, threads, 0, s>>>(
          kind, (const uint16_t*)in, in_ld, (uint16_t*)out, out_rows, out_cols, out_ld, alpha,
          alpha_out, lrows, lcols);
      break;
    case 4:
      transform_kernel<uint32_t><<<(unsigned)blocks, threads, 0, s>>>(
          kind, (const uint32_t*)in, in_ld, (uint32_t*)out, out_rows, out_cols, out_ld, alpha,
          alpha_out, lrows, lcols);
      break;
    case 8:
      transform_kernel<uint64_t><<<(unsigned)blocks, threads, 0, s>>>(
          kind, (const uint64_t*)in, in_ld, (uint64_t*)out, out_rows, out_cols, out_ld, alpha,
          alpha_out, lrows, lcols);
      break;
    default:
      return fail(TPP_E_SPEC_DTYPE, "transform: unsupported element size");
  }
  TPP_CUDA_LAUNCH_CHECK("transform_kernel");
  return TPP_OK;
}

}  // namespace tpp

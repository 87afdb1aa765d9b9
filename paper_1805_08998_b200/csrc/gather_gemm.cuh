// Row-gathered GEMM on the FP64 tensor cores, for the implicit (sketch-only) route of the
// large far blocks: their T = sum_t L_t R_t^T is never materialized, only applied,
//   Z = [R_1 .. R_T]^T Omega      (every row of Z is one column of some R_t)
//   W = [L_1 .. L_T]^T Q_Y        (every row of W is one column of some L_t)
// The rows of one 64-row output tile come from several factors (ranks ~10-50 each) but
// share the K range, so the A tile is gathered row by row -- each row one contiguous
// vector of the factor pool -- and the tensor cores see one dense 64 x 64 x K product
// instead of one under-filled product per factor.
//
//   out(r, j) = sum_kk A_r[kk] * B[kk + j * b_ld],  r < rows, j < cols, kk < klen
//   A_r[kk] = bufs[seg.buf][seg.off + x * seg.ld + kk - seg.kb]  for kk in [seg.kb, seg.ke)
//   (zero elsewhere) for the x-th row of the segment holding r: rows with different K
//   ranges (terms created on sub-blocks) share a tile, each zero-filled outside its range.
#pragma once
#include <cstdint>

#include "gemm.cuh"

namespace hx {

struct GSeg {
  int64_t off;
  int32_t ld;
  int16_t rows;
  uint8_t buf, pad;
  int32_t kb, ke;  // valid K range of the segment's rows, tile coordinates
};
static_assert(sizeof(GSeg) == 24, "GSeg layout");

struct GTile {
  int64_t out_off, b_off;
  int32_t out_ld, b_ld;
  int32_t seg_begin, seg_end;
  int32_t klen;
  int16_t rows, cols;
  uint8_t out_buf, b_buf, pad[6];
};
static_assert(sizeof(GTile) == 48, "GTile layout");

// Stage KC k-slots of a 64-row operand whose rows are contiguous vectors: smem [row][slot].
// Row r holds rowp[r][kk] for kk in [kb[r], ke[r]) (rowp already shifted by -kb[r]).
template <class C>
__device__ __forceinline__ void stage_rows(unsigned sbase, const double* const* rowp,
                                           const int* kb, const int* ke, const double* safe,
                                           int nrows, int kk0) {
  constexpr int PK = C::KC / 2, RL = C::THREADS / PK;
  const int tid = threadIdx.x;
  const int q = tid % PK, r0 = tid / PK;
  const int kk = kk0 + 2 * q;
#pragma unroll 2
  for (int r = r0; r < C::TM; r += RL) {
    const unsigned dst = sbase + 8u * unsigned(r * C::LDK + 2 * q);
    bool v0 = false, v1 = false;
    const double* src = safe;
    if (r < nrows) {
      v0 = kk >= kb[r] && kk < ke[r];
      v1 = kk + 1 >= kb[r] && kk + 1 < ke[r];
      src = rowp[r] + kk;
    }
    if (v0 && v1 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
      cp_async16(dst, src, 16);
    } else {
      cp_async8(dst, v0 ? src : safe, v0 ? 8 : 0);
      cp_async8(dst + 8u, v1 ? src + 1 : safe, v1 ? 8 : 0);
    }
  }
}

template <class C>
__global__ void __launch_bounds__(C::THREADS) gather_gemm_kernel(
    const GTile* __restrict__ tiles, const GSeg* __restrict__ segs,
    const __grid_constant__ BufPtrs bufs, int n_tiles) {
  extern __shared__ __align__(16) double smem[];
  __shared__ const double* arow[C::TM];
  __shared__ const double* brow[C::TM];
  __shared__ int akb[C::TM], ake[C::TM], bkb[C::TM], bke[C::TM];
  if (int(blockIdx.x) >= n_tiles) return;
  const GTile tl = tiles[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  if (threadIdx.x == 0) {
    int r = 0;
    for (int s = tl.seg_begin; s < tl.seg_end; ++s) {
      const GSeg sg = segs[s];
      const double* base = bufs.p[sg.buf] + sg.off;
      for (int x = 0; x < sg.rows && r < C::TM; ++x) {
        akb[r] = sg.kb;
        ake[r] = sg.ke;
        arow[r++] = base + int64_t(x) * sg.ld - sg.kb;
      }
    }
  }
  if (threadIdx.x < C::TM) {
    const double* B = bufs.p[tl.b_buf] + tl.b_off;
    brow[threadIdx.x] = B + int64_t(threadIdx.x) * tl.b_ld;
    bkb[threadIdx.x] = 0;
    bke[threadIdx.x] = tl.klen;
  }
  __syncthreads();
  const double* safe = bufs.p[tl.b_buf] + tl.b_off;

  double acc[C::FR][C::FR][2];
#pragma unroll
  for (int a = 0; a < C::FR; ++a)
#pragma unroll
    for (int b = 0; b < C::FR; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  Chunk ch;
  ch.akc = ch.bkc = 1;
  ch.amask = ch.bmask = 0;
#pragma unroll
  for (int a = 0; a < C::FR; ++a) {
    if (wm * C::WT + a * 8 < tl.rows) ch.amask |= 1u << a;
    if (wn * C::WT + a * 8 < tl.cols) ch.bmask |= 1u << a;
  }
  const int nch = (tl.klen + C::KC - 1) / C::KC;
  auto stage = [&](int st, int c) {
    double* sP = smem + st * C::STAGE;
    const unsigned sp = static_cast<unsigned>(__cvta_generic_to_shared(sP));
    const unsigned sq = static_cast<unsigned>(__cvta_generic_to_shared(sP + C::OPSZ));
    stage_rows<C>(sp, arow, akb, ake, safe, tl.rows, c * C::KC);
    stage_rows<C>(sq, brow, bkb, bke, safe, tl.cols, c * C::KC);
  };
  if (nch > 0) stage(0, 0);
  cp_async_commit();
  for (int c = 0; c < nch; ++c) {
    if (c + 1 < nch) stage((c + 1) & 1, c + 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* sP = smem + (c & 1) * C::STAGE;
    ch.used = min(C::KC, tl.klen - c * C::KC);
    if (ch.amask && ch.bmask) mma_chunk_t<C, 1, 1>(acc, sP, sP + C::OPSZ, ch, wm, wn, lane);
    __syncthreads();
  }
  cp_async_wait<0>();
  double* out = bufs.p[tl.out_buf] + tl.out_off;
#pragma unroll
  for (int a = 0; a < C::FR; ++a) {
    const int r = wm * C::WT + a * 8 + (lane >> 2);
#pragma unroll
    for (int b = 0; b < C::FR; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = wn * C::WT + b * 8 + (lane & 3) * 2 + h;
        if (r < tl.rows && cc < tl.cols) out[r + int64_t(cc) * tl.out_ld] = acc[a][b][h];
      }
  }
}

}  // namespace hx

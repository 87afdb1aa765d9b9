// Grouped sum-of-products GEMM on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64).
//
// One CTA computes one Tile: out[rows x cols] (=|+=) sum over the tile's groups, over each
// group's terms, of P_t(tile rows, :) * Q_t(:, tile cols)  (layouts in hx_types.h).
// This single kernel runs every contraction of the product:
//   * k x k cores            V_A^T U_B                        (_thin_product, sumexpr.py:99-107)
//   * pushed-through factors V_B core^T, U_A core, X U_B, X^T V_A (sumexpr.py:103-117,
//                            hmatrix.py:177-202)
//   * block materialization  sum_j U_j V_j^T + sum_p D_A D_B  (SumExpression.apply_mat,
//                            sumexpr.py:59-66; evaluate_dense, sumexpr.py:165-170)
//   * sketch products        T Omega, T^T Q                   (recompression)
//
// TM x TM tile, 4 warps in a 2 x 2 grid; a warp owns (TM/2) x (TM/2) as (TM/16)^2 DMMA
// 8x8 accumulators.  K is streamed in chunks of KC through double-buffered shared memory
// filled with cp.async (8-byte, zero-filled outside the term's extent), so the next
// chunk -- possibly of the next term -- loads while the current one multiplies.
#pragma once
#include <cstdint>

#include "hx_types.h"

namespace hx {

struct BufPtrs {
  double* p[NUM_BUFS];
};

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int TM>
struct GemmCfg {
  static constexpr int KC = 16;            // k chunk
  static constexpr int LDS = TM + 4;       // padded smem row (doubles): 2-way max on DMMA reads
  static constexpr int WT = TM / 2;        // warp tile side
  static constexpr int FR = WT / 8;        // 8x8 fragments per warp side
  static constexpr int THREADS = 128;
  static constexpr int STAGE = 2 * KC * LDS;  // P + Q chunk (doubles)
};

// Cursor over the (group, term, k-chunk) sequence of one tile.
struct ChunkCursor {
  int g, g_end, t, t_end, k0;
};

template <int TM>
__device__ __forceinline__ void load_chunk(double* __restrict__ sP, double* __restrict__ sQ,
                                           const BufPtrs& bufs, const Term& tm, int k0,
                                           int row0, int col0, int tile_rows, int tile_cols) {
  using C = GemmCfg<TM>;
  const int tid = threadIdx.x;
  const double* A = bufs.p[tm.a_buf] + tm.a_off;
  const double* B = bufs.p[tm.b_buf] + tm.b_off;
  const int i0 = row0 - tm.r_lo;   // first term row of this tile
  const int j0 = col0 - tm.c_lo;
  const int kr = tm.k - k0;         // remaining k
  // P chunk: TM rows x KC
  if (tm.a_kc == 0) {
#pragma unroll
    for (int e = tid; e < TM * C::KC; e += C::THREADS) {
      const int i = e % TM, kk = e / TM;
      const int gi = i0 + i;
      const bool v = (i < tile_rows) && (gi >= 0) && (gi < tm.rows) && (kk < kr);
      const double* src = v ? A + gi + int64_t(k0 + kk) * tm.a_ld : A;
      cp_async8(sP + kk * C::LDS + i, src, v);
    }
  } else {
#pragma unroll
    for (int e = tid; e < TM * C::KC; e += C::THREADS) {
      const int kk = e % C::KC, i = e / C::KC;
      const int gi = i0 + i;
      const bool v = (i < tile_rows) && (gi >= 0) && (gi < tm.rows) && (kk < kr);
      const double* src = v ? A + (k0 + kk) + int64_t(gi) * tm.a_ld : A;
      cp_async8(sP + kk * C::LDS + i, src, v);
    }
  }
  // Q chunk: KC x TM cols
  if (tm.b_kc == 0) {
#pragma unroll
    for (int e = tid; e < TM * C::KC; e += C::THREADS) {
      const int j = e % TM, kk = e / TM;
      const int gj = j0 + j;
      const bool v = (j < tile_cols) && (gj >= 0) && (gj < tm.cols) && (kk < kr);
      const double* src = v ? B + gj + int64_t(k0 + kk) * tm.b_ld : B;
      cp_async8(sQ + kk * C::LDS + j, src, v);
    }
  } else {
#pragma unroll
    for (int e = tid; e < TM * C::KC; e += C::THREADS) {
      const int kk = e % C::KC, j = e / C::KC;
      const int gj = j0 + j;
      const bool v = (j < tile_cols) && (gj >= 0) && (gj < tm.cols) && (kk < kr);
      const double* src = v ? B + (k0 + kk) + int64_t(gj) * tm.b_ld : B;
      cp_async8(sQ + kk * C::LDS + j, src, v);
    }
  }
}

// Advance the cursor to the next non-empty chunk; returns false at the end.
__device__ __forceinline__ bool next_chunk(ChunkCursor& c, const Group* __restrict__ groups,
                                           const Term* __restrict__ terms, int KC, Term& tm) {
  while (true) {
    if (c.t < c.t_end) {
      if (c.k0 < tm.k) return true;
      ++c.t;
      c.k0 = 0;
      if (c.t < c.t_end) {
        tm = terms[c.t];
        continue;
      }
    }
    ++c.g;
    if (c.g >= c.g_end) return false;
    const Group gr = groups[c.g];
    c.t = gr.t_begin;
    c.t_end = gr.t_end;
    c.k0 = 0;
    if (c.t < c.t_end) tm = terms[c.t];
  }
}

template <int TM>
__global__ void __launch_bounds__(128) grouped_gemm_kernel(const Tile* __restrict__ tiles,
                                                           const Group* __restrict__ groups,
                                                           const Term* __restrict__ terms,
                                                           const __grid_constant__ BufPtrs bufs,
                                                           double* __restrict__ sumsq,
                                                           int n_tiles) {
  using C = GemmCfg<TM>;
  __shared__ __align__(16) double smem[2 * C::STAGE];
  __shared__ double red[4];
  const int tile_idx = blockIdx.x;
  if (tile_idx >= n_tiles) return;
  const Tile tl = tiles[tile_idx];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1;

  double acc[C::FR][C::FR][2];
#pragma unroll
  for (int a = 0; a < C::FR; ++a)
#pragma unroll
    for (int b = 0; b < C::FR; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // two cursors: `ld` runs one chunk ahead of `cm` (the chunk being multiplied)
  ChunkCursor ld{tl.g_begin - 1, tl.g_end, 0, 0, 0};
  Term tld;
  tld.k = 0;
  bool have = next_chunk(ld, groups, terms, C::KC, tld);
  int stage = 0;
  if (have) {
    load_chunk<TM>(smem, smem + C::KC * C::LDS, bufs, tld, ld.k0, tl.row0, tl.col0, tl.rows,
                   tl.cols);
  }
  cp_async_commit();
  while (have) {
    const int kcur = min(C::KC, tld.k - ld.k0);
    // 8x8 fragments of this warp that the current term touches (terms created on a
    // sub-block, or stacked cores, cover only part of the tile): skip the others
    unsigned amask = 0, bmask = 0;
    {
      const int ra = tld.r_lo - tl.row0, rb = ra + tld.rows;
      const int ca = tld.c_lo - tl.col0, cb = ca + tld.cols;
#pragma unroll
      for (int a = 0; a < C::FR; ++a) {
        const int f0 = wm * C::WT + a * 8;
        if (f0 < rb && f0 + 8 > ra) amask |= 1u << a;
        const int g0 = wn * C::WT + a * 8;
        if (g0 < cb && g0 + 8 > ca) bmask |= 1u << a;
      }
    }
    // prefetch the following chunk into the other stage
    ld.k0 += C::KC;
    bool more = next_chunk(ld, groups, terms, C::KC, tld);
    if (more) {
      double* s = smem + (stage ^ 1) * C::STAGE;
      load_chunk<TM>(s, s + C::KC * C::LDS, bufs, tld, ld.k0, tl.row0, tl.col0, tl.rows,
                     tl.cols);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* sP = smem + stage * C::STAGE;
    const double* sQ = sP + C::KC * C::LDS;
    const int ksteps = (kcur + 3) >> 2;
    if (amask && bmask) {
      const bool full = amask == (1u << C::FR) - 1 && bmask == (1u << C::FR) - 1;
      for (int ks = 0; ks < ksteps; ++ks) {
        const int kk = ks * 4 + (lane & 3);
        double af[C::FR], bf[C::FR];
#pragma unroll
        for (int a = 0; a < C::FR; ++a)
          af[a] = sP[kk * C::LDS + wm * C::WT + a * 8 + (lane >> 2)];
#pragma unroll
        for (int b = 0; b < C::FR; ++b)
          bf[b] = sQ[kk * C::LDS + wn * C::WT + b * 8 + (lane >> 2)];
        if (full) {
#pragma unroll
          for (int a = 0; a < C::FR; ++a)
#pragma unroll
            for (int b = 0; b < C::FR; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        } else {
#pragma unroll
          for (int a = 0; a < C::FR; ++a)
#pragma unroll
            for (int b = 0; b < C::FR; ++b)
              if ((amask >> a) & (bmask >> b) & 1u)
                dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
      }
    }
    __syncthreads();
    stage ^= 1;
    have = more;
  }
  cp_async_wait<0>();

  // epilogue
  double* out = bufs.p[tl.out_buf] + tl.out_off;
  double ss = 0.0;
#pragma unroll
  for (int a = 0; a < C::FR; ++a) {
    const int r = wm * C::WT + a * 8 + (lane >> 2);
#pragma unroll
    for (int b = 0; b < C::FR; ++b) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = wn * C::WT + b * 8 + (lane & 3) * 2 + h;
        if (r < tl.rows && c < tl.cols) {
          double* dst = out + r + int64_t(c) * tl.out_ld;
          double v = acc[a][b][h];
          if (tl.mode == MODE_ADD) v += *dst;
          *dst = v;
          ss += v * v;
        }
      }
    }
  }
  if (tl.mode == MODE_STORE_SUMSQ) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (threadIdx.x == 0) sumsq[tl.aux] = (red[0] + red[1]) + (red[2] + red[3]);
  }
}

}  // namespace hx

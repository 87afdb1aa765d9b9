// Grouped sum-of-products GEMM on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64).
//
// One CTA computes one Tile: out[rows x cols] (=|+=) sum over the tile's groups, over each
// group's terms, of P_t(tile rows, :) * Q_t(:, tile cols)  (layouts in hx_types.h).
// This single kernel runs every contraction of the product:
//   * stacked k x k cores    V_l^T G, U_l^T G                 (_thin_product, sumexpr.py:99-107)
//   * pushed-through factors X G, X^T G                       (sumexpr.py:103-117,
//                            hmatrix.py:177-202)
//   * block materialization  sum_j U_j V_j^T + sum_p D_A D_B  (SumExpression.apply_mat,
//                            sumexpr.py:59-66; evaluate_dense, sumexpr.py:165-170)
//   * sketch products        T Omega, T^T Q                   (recompression)
//
// TM x TM tile, 4 warps (2 x 2); a warp owns (TM/2)^2 as 8x8 DMMA accumulators.
// Terms of the product have small k (ranks ~10-50), so K is streamed in chunks of KC = 32
// "slots" that pack consecutive terms: a chunk is a list of segments (term, k offset,
// slot count) with one staging layout.  Each operand is staged in the layout it has in HBM
// so that copies are 16-byte cp.async where aligned: tile-contiguous operands as
// [slot][tile index], k-contiguous ones as [tile index][slot].  Rows outside a term's
// extent are zero-filled by the copies (src-size 0); unused pad slots are zeroed.  The
// double-buffered chunk ring overlaps the next chunk's copies with the current DMMAs.
#pragma once
#include <cstdint>

#include "hx_types.h"

#ifndef HX_ZERO_MASKED
#define HX_ZERO_MASKED 1  // 0: predicate each DMMA on its fragment mask instead
#endif

namespace hx {

struct BufPtrs {
  double* p[NUM_BUFS];
};

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(unsigned saddr, const void* gmem, int valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(valid));
}
__device__ __forceinline__ void cp_async8(unsigned saddr, const void* gmem, int valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(valid));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int TM_, int KC_ = 32, int MINB_ = 1>
struct GemmCfg {
  static constexpr int TM = TM_;
  static constexpr int KC = KC_;               // slots per chunk
  static constexpr int MINB = MINB_;           // resident CTAs per SM to budget registers for
  static constexpr int LDI = TM + 4;           // [slot][i] row (doubles), 16B aligned
  static constexpr int LDK = KC + 4;           // [i][slot] row (doubles), 16B aligned
  static constexpr int OPSZ = (KC * LDI > TM * LDK) ? KC * LDI : TM * LDK;
  static constexpr int WT = TM / 2;            // warp tile side
  static constexpr int FR = WT / 8;            // 8x8 fragments per warp side
  static constexpr int THREADS = 128;
  static constexpr int STAGE = 2 * OPSZ;       // P + Q (doubles)
  static constexpr int SMEM = 2 * STAGE * 8;
  static constexpr int MAXSEG = 8;
};

using Gemm64 = GemmCfg<64, 32, 3>;
using Gemm32 = GemmCfg<32>;
// short-K batches (stacked cores, X G bands: K ~ 70): half-size chunks, 41 KB of smem and
// <= 128 registers, so four CTAs share an SM and hide each other's tile prologues
using Gemm64s = GemmCfg<64, 16, 4>;

// Cursor over (group, term, k offset) of one tile.
struct Cursor {
  int g, g_end, t, t_end, k0;
  Term tm;
};

struct Chunk {
  int used;              // slots filled (0 = no chunk)
  int akc, bkc;          // staged layouts of P and Q
  unsigned amask, bmask; // 8x8 fragments of this warp touched by any segment
};

// Advance to the next term with k > 0 (c.k0 reset); false at the end of the tile.
__device__ __forceinline__ bool next_term(Cursor& c, const Group* __restrict__ groups,
                                          const Term* __restrict__ terms) {
  while (true) {
    ++c.t;
    if (c.t < c.t_end) {
      c.tm = terms[c.t];
      c.k0 = 0;
      if (c.tm.k > 0) return true;
      continue;
    }
    ++c.g;
    if (c.g >= c.g_end) return false;
    const Group gr = groups[c.g];
    c.t = gr.t_begin - 1;
    c.t_end = gr.t_end;
  }
}

// Stage n slots of one operand of one segment.
//   kc == 0: X(idx, kk) = base[idx + kk*ld] -> smem [slot][idx] (LDI)
//   kc == 1: X(idx, kk) = base[kk + idx*ld] -> smem [idx][slot] (LDK)
// base points at tile index 0, k offset of the segment.  idx valid in [lo, hi).
template <class C>
__device__ __forceinline__ void stage_seg(unsigned sbase, const double* base,
                                          const double* safe, int ld, int kc,
                                          int lo, int hi, int slot0, int n) {
  constexpr int TM = C::TM;
  const int tid = threadIdx.x;
  if (kc == 0) {
    const bool al = ((reinterpret_cast<uintptr_t>(base) & 15) == 0) && ((ld & 1) == 0) &&
                    (((lo | hi) & 1) == 0);
    if (al) {
      // thread -> row pair p, slot lane c; TM/2 pairs per slot column
      constexpr int PR = TM / 2, CL = C::THREADS / PR;
      const int p = tid % PR, c = tid / PR;
      const int i = 2 * p;
      const int v = (i >= lo && i < hi) ? 16 : 0;
      const double* src = base + i + int64_t(c) * ld;
      unsigned dst = sbase + 8u * unsigned((slot0 + c) * C::LDI + i);
      const int64_t step = int64_t(CL) * ld;
      for (int s = c; s < n; s += CL) {
        cp_async16(dst, v ? src : safe, v);
        src += step;
        dst += 8u * CL * C::LDI;
      }
    } else {
      const int i = tid % TM, c = tid / TM;
      constexpr int CL = C::THREADS / TM;
      const int v = (i >= lo && i < hi) ? 8 : 0;
      const double* src = base + i + int64_t(c) * ld;
      unsigned dst = sbase + 8u * unsigned((slot0 + c) * C::LDI + i);
      for (int s = c; s < n; s += CL) {
        cp_async8(dst, v ? src : safe, v);
        src += int64_t(CL) * ld;
        dst += 8u * CL * C::LDI;
      }
    }
  } else {
    const bool al = ((reinterpret_cast<uintptr_t>(base) & 15) == 0) && ((ld & 1) == 0) &&
                    ((slot0 & 1) == 0);
    if (al) {
      // thread -> slot pair q, row lane r: pairs along k
      constexpr int PK = C::KC / 2, RL = C::THREADS / PK;
      const int q = tid % PK, r = tid / PK;
      const int kk = 2 * q;
      if (kk < n) {
        // an odd segment end is copied alone: a zero-filled pair half would clobber the
        // first slot of the next segment
        const bool pair = kk + 1 < n;
        const double* src = base + kk + int64_t(r) * ld;
        unsigned dst = sbase + 8u * unsigned(r * C::LDK + slot0 + kk);
        for (int i = r; i < TM; i += RL) {
          const bool v = i >= lo && i < hi;
          if (pair) cp_async16(dst, v ? src : safe, v ? 16 : 0);
          else cp_async8(dst, v ? src : safe, v ? 8 : 0);
          src += int64_t(RL) * ld;
          dst += 8u * RL * C::LDK;
        }
      }
    } else {
      constexpr int RL = C::THREADS / C::KC;
      const int kk = tid % C::KC, r = tid / C::KC;
      if (kk < n) {
        const double* src = base + kk + int64_t(r) * ld;
        unsigned dst = sbase + 8u * unsigned(r * C::LDK + slot0 + kk);
        for (int i = r; i < TM; i += RL) {
          const bool v = i >= lo && i < hi;
          cp_async8(dst, v ? src : safe, v ? 8 : 0);
          src += int64_t(RL) * ld;
          dst += 8u * RL * C::LDK;
        }
      }
    }
  }
}

// Stage n slots of a column-gathered operand (Term b_kc == 2): X(idx, kk) =
// colp[idx][off + kk] -> smem [idx][slot] (LDK); idx valid in [lo, hi).
template <class C>
__device__ __forceinline__ void stage_cols(unsigned sbase, const double* const* colp, int64_t off,
                                           const double* safe, int lo, int hi, int slot0, int n) {
  constexpr int PK = C::KC / 2, RL = C::THREADS / PK;
  const int tid = threadIdx.x;
  const int q = tid % PK, r = tid / PK;
  const int kk = 2 * q;
  if (kk >= n) return;
  const bool pair = kk + 1 < n;
  for (int i = r; i < C::TM; i += RL) {
    const bool v = i >= lo && i < hi;
    const unsigned dst = sbase + 8u * unsigned(i * C::LDK + slot0 + kk);
    const double* src = v ? colp[i] + off + kk : safe;
    if (pair && v && ((slot0 & 1) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
      cp_async16(dst, src, 16);
    } else {
      cp_async8(dst, src, v ? 8 : 0);
      if (pair) cp_async8(dst + 8u, v ? src + 1 : safe, v ? 8 : 0);
    }
  }
}

// Zero slots [a, b) of an operand in either layout (pad up to a multiple of 4).
template <class C>
__device__ __forceinline__ void zero_slots(double* s, int kc, int a, int b) {
  const int n = b - a;
  if (n <= 0) return;
  for (int e = threadIdx.x; e < n * C::TM; e += C::THREADS) {
    const int kk = a + e / C::TM, i = e % C::TM;
    s[kc ? i * C::LDK + kk : kk * C::LDI + i] = 0.0;
  }
}

// Fill one chunk from the cursor.  Returns the chunk descriptor (used = 0: nothing left).
template <class C>
__device__ __forceinline__ Chunk build_chunk(double* sP, double* sQ, Cursor& cur, bool& have,
                                             const Group* __restrict__ groups,
                                             const Term* __restrict__ terms,
                                             const BufPtrs& bufs, const Tile& tl, int wm, int wn,
                                             const double* const* colp) {
  Chunk ch;
  ch.used = 0;
  ch.amask = ch.bmask = 0;
  ch.akc = cur.tm.a_kc;
  ch.bkc = cur.tm.b_kc ? 1 : 0;  // smem layout: column-gathered operands stage like kc 1
  const unsigned sp = static_cast<unsigned>(__cvta_generic_to_shared(sP));
  const unsigned sq = static_cast<unsigned>(__cvta_generic_to_shared(sQ));
  int nseg = 0;
  while (have && ch.used < C::KC && nseg < C::MAXSEG) {
    const Term& tm = cur.tm;
    if (tm.a_kc != ch.akc || (tm.b_kc ? 1 : 0) != ch.bkc) break;  // one layout per chunk
    const int n = min(C::KC - ch.used, tm.k - cur.k0);
    const int i0 = tl.row0 - tm.r_lo, j0 = tl.col0 - tm.c_lo;
    const int rlo = max(0, -i0), rhi = min(int(tl.rows), tm.rows - i0);
    const int clo = max(0, -j0), chi = min(int(tl.cols), tm.cols - j0);
    const double* A = bufs.p[tm.a_buf] + tm.a_off;
    const double* B = bufs.p[tm.b_buf] + tm.b_off;
    const double* pa =
        tm.a_kc ? A + cur.k0 + int64_t(i0) * tm.a_ld : A + i0 + int64_t(cur.k0) * tm.a_ld;
    const double* pb =
        tm.b_kc ? B + cur.k0 + int64_t(j0) * tm.b_ld : B + j0 + int64_t(cur.k0) * tm.b_ld;
    // masked copies read nothing, but get an in-bounds address (the term's first element)
    stage_seg<C>(sp, pa, A, tm.a_ld, tm.a_kc, rlo, rhi, ch.used, n);
    if (tm.b_kc == 2)
      stage_cols<C>(sq, colp, tm.b_off + cur.k0, bufs.p[BUF_A], clo, chi, ch.used, n);
    else
      stage_seg<C>(sq, pb, B, tm.b_ld, tm.b_kc, clo, chi, ch.used, n);
#pragma unroll
    for (int a = 0; a < C::FR; ++a) {
      const int f0 = wm * C::WT + a * 8;
      if (f0 < rhi && f0 + 8 > rlo) ch.amask |= 1u << a;
      const int g0 = wn * C::WT + a * 8;
      if (g0 < chi && g0 + 8 > clo) ch.bmask |= 1u << a;
    }
    ch.used += n;
    ++nseg;
    cur.k0 += n;
    if (cur.k0 >= tm.k) have = next_term(cur, groups, terms);
  }
  const int padded = (ch.used + 3) & ~3;
  zero_slots<C>(sP, ch.akc, ch.used, padded);
  zero_slots<C>(sQ, ch.bkc, ch.used, padded);
  return ch;
}

// DMMA over one staged chunk; AK/BK: compile-time staging layouts.
template <class C, int AK, int BK>
__device__ __forceinline__ void mma_chunk_t(double (&acc)[C::FR][C::FR][2], const double* sP,
                                            const double* sQ, const Chunk& ch, int wm, int wn,
                                            int lane) {
  constexpr int SA_I = AK ? C::LDK : 1, SA_K = AK ? 1 : C::LDI;
  constexpr int SB_I = BK ? C::LDK : 1, SB_K = BK ? 1 : C::LDI;
  const int ksteps = (ch.used + 3) >> 2;
  const int r = lane >> 2, q = lane & 3;
  const double* pa = sP + (wm * C::WT + r) * SA_I + q * SA_K;
  const double* pb = sQ + (wn * C::WT + r) * SB_I + q * SB_K;
  const bool full = ch.amask == (1u << C::FR) - 1 && ch.bmask == (1u << C::FR) - 1;
  if (full) {
    for (int ks = 0; ks < ksteps; ++ks) {
      double af[C::FR], bf[C::FR];
#pragma unroll
      for (int a = 0; a < C::FR; ++a) af[a] = pa[a * 8 * SA_I + ks * 4 * SA_K];
#pragma unroll
      for (int b = 0; b < C::FR; ++b) bf[b] = pb[b * 8 * SB_I + ks * 4 * SB_K];
#pragma unroll
      for (int a = 0; a < C::FR; ++a)
#pragma unroll
        for (int b = 0; b < C::FR; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  } else {
#if HX_ZERO_MASKED
    // untouched fragments multiply staged zeros (rows outside every segment are zero-
    // filled by the copies): every DMMA is unconditional, with no per-instruction warp
    // re-convergence, at the cost of the masked fragments' DMMA slots (config 2
    // formation 120 -> 114 ms)
    for (int ks = 0; ks < ksteps; ++ks) {
      double af[C::FR], bf[C::FR];
#pragma unroll
      for (int a = 0; a < C::FR; ++a) af[a] = pa[a * 8 * SA_I + ks * 4 * SA_K];
#pragma unroll
      for (int b = 0; b < C::FR; ++b) bf[b] = pb[b * 8 * SB_I + ks * 4 * SB_K];
#pragma unroll
      for (int a = 0; a < C::FR; ++a)
#pragma unroll
        for (int b = 0; b < C::FR; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
#else
    for (int ks = 0; ks < ksteps; ++ks) {
      double af[C::FR], bf[C::FR];
#pragma unroll
      for (int a = 0; a < C::FR; ++a) af[a] = pa[a * 8 * SA_I + ks * 4 * SA_K];
#pragma unroll
      for (int b = 0; b < C::FR; ++b) bf[b] = pb[b * 8 * SB_I + ks * 4 * SB_K];
#pragma unroll
      for (int a = 0; a < C::FR; ++a)
#pragma unroll
        for (int b = 0; b < C::FR; ++b)
          if ((ch.amask >> a) & (ch.bmask >> b) & 1u)
            dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
#endif
  }
}

template <class C>
__device__ __forceinline__ void mma_chunk(double (&acc)[C::FR][C::FR][2], const double* sP,
                                          const double* sQ, const Chunk& ch, int wm, int wn,
                                          int lane) {
  if (!(ch.amask && ch.bmask)) return;
  switch (ch.akc * 2 + ch.bkc) {
    case 0: mma_chunk_t<C, 0, 0>(acc, sP, sQ, ch, wm, wn, lane); break;
    case 1: mma_chunk_t<C, 0, 1>(acc, sP, sQ, ch, wm, wn, lane); break;
    case 2: mma_chunk_t<C, 1, 0>(acc, sP, sQ, ch, wm, wn, lane); break;
    default: mma_chunk_t<C, 1, 1>(acc, sP, sQ, ch, wm, wn, lane); break;
  }
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB) grouped_gemm_kernel(
    const Tile* __restrict__ tiles, const Group* __restrict__ groups,
    const Term* __restrict__ terms, const __grid_constant__ BufPtrs bufs,
    double* __restrict__ sumsq, int n_tiles, const ColRec* __restrict__ gcols) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double red[C::THREADS / 32];
  __shared__ const double* colp[C::TM];
  const int tile_idx = blockIdx.x;
  if (tile_idx >= n_tiles) return;
  const Tile tl = tiles[tile_idx];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  if (tl.mode == MODE_GCOL) {
    // column pointers of the tile's slice of the virtual matrix G
    if (int(threadIdx.x) < tl.cols) {
      const int j = tl.col0 + threadIdx.x;
      int idx = tl.aux;
      ColRec r = gcols[idx];
      while (j >= r.col + r.k) r = gcols[++idx];
      colp[threadIdx.x] = bufs.p[r.buf] + r.src_off + int64_t(j - r.col) * r.ld;
    }
    __syncthreads();
  }

  double acc[C::FR][C::FR][2];
#pragma unroll
  for (int a = 0; a < C::FR; ++a)
#pragma unroll
    for (int b = 0; b < C::FR; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  Cursor cur;
  cur.g = tl.g_begin - 1;
  cur.g_end = tl.g_end;
  cur.t = cur.t_end = 0;
  cur.k0 = 0;
  bool have = next_term(cur, groups, terms);
  int stage = 0;
  Chunk now =
      build_chunk<C>(smem, smem + C::OPSZ, cur, have, groups, terms, bufs, tl, wm, wn, colp);
  cp_async_commit();
  while (now.used > 0) {
    double* ns = smem + (stage ^ 1) * C::STAGE;
    Chunk nxt =
        build_chunk<C>(ns, ns + C::OPSZ, cur, have, groups, terms, bufs, tl, wm, wn, colp);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double* sP = smem + stage * C::STAGE;
    mma_chunk<C>(acc, sP, sP + C::OPSZ, now, wm, wn, lane);
    __syncthreads();
    stage ^= 1;
    now = nxt;
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
          if (tl.mode == MODE_RESID_SUMSQ) {
            v = *dst - v;  // residual of the tile against its approximation; not stored
          } else {
            if (tl.mode == MODE_ADD) v += *dst;
            *dst = v;
          }
          ss += v * v;
        }
      }
    }
  }
  if (tl.mode == MODE_STORE_SUMSQ || tl.mode == MODE_RESID_SUMSQ) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < C::THREADS / 32; ++w) t += red[w];
      sumsq[tl.aux] = t;
    }
  }
}

}  // namespace hx

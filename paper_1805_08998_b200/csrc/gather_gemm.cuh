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
#include "gemm_ws.cuh"

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

// ---------------------------------------------------------------------------------------
// Warp-specialized, persistent version (the structure of gemm_ws.cuh).  The sketch products
// are thin (cols = the sketch width, 16-64) and long (K = the block dimension), so the
// kernel is bound by streaming the gathered A rows: 2 producer warps keep a 3-deep ring of
// 32-slot chunks in flight per CTA with cp.async (no CTA barrier in the main loop), rows and
// columns beyond the tile's 8-aligned extent are not staged at all, and the 4 consumer
// warps split the tile by rows (16 each) so that all of them work whatever the width.
struct GwsDesc {
  int32_t used, last;
};

template <class C>
__device__ __forceinline__ void gws_stage(unsigned sbase, const double* const* rowp,
                                          const int* kb, const int* ke, const double* safe,
                                          int nrows, int nrows8, int kk0, bool fast, int tid) {
  constexpr int PK = C::KC / 2, RL = C::NPT / PK;
  const int q = tid % PK, r0 = tid / PK;
  const int kk = kk0 + 2 * q;
  unsigned dst = sbase + 8u * unsigned(r0 * C::LDK + 2 * q);
  if (fast) {
    // every row covers the chunk and is 16-byte aligned, or is a zero row
#pragma unroll 4
    for (int r = r0; r < nrows8; r += RL) {
      const double* p = r < nrows ? rowp[r] : nullptr;  // nullptr: a zero (pad) row
      cp_async16(dst, p ? p + kk : safe, p ? 16 : 0);
      dst += 8u * RL * C::LDK;
    }
    return;
  }
  for (int r = r0; r < nrows8; r += RL) {
    bool v0 = false, v1 = false;
    const double* src = safe;
    if (r < nrows && rowp[r] != nullptr) {
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
    dst += 8u * RL * C::LDK;
  }
}

// consumer warp cw: rows [16 cw, 16 cw + 16) x NFC column fragments
template <class C, int NFC>
__device__ __forceinline__ void gws_mma(double (&acc)[2][8][2], const double* sP,
                                        const double* sQ, int used, int cw, int lane,
                                        unsigned amask) {
  const int ksteps = (used + 3) >> 2;
  const int r = lane >> 2, q = lane & 3;
  const double* pa = sP + (cw * 16 + r) * C::LDK + q;
  const double* pb = sQ + r * C::LDK + q;
  for (int ks = 0; ks < ksteps; ++ks) {
    double af[2], bf[NFC];
#pragma unroll
    for (int a = 0; a < 2; ++a) af[a] = (amask >> a) & 1u ? pa[a * 8 * C::LDK + ks * 4] : 0.0;
#pragma unroll
    for (int b = 0; b < NFC; ++b) bf[b] = pb[b * 8 * C::LDK + ks * 4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < NFC; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
  }
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB) gather_gemm_ws_kernel(
    const GTile* __restrict__ tiles, const GSeg* __restrict__ segs,
    const __grid_constant__ BufPtrs bufs, int n_tiles) {
  static_assert(C::NPW == 2 && C::NCW == 4 && C::TM == 64,
                "warp 0 builds the A row table, warp 1 the B table; 4 consumers x 16 rows");
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES];
  __shared__ GwsDesc desc[C::STAGES];
  __shared__ const double* arow[C::TM];
  __shared__ const double* brow[C::TM];
  __shared__ int akb[C::TM], ake[C::TM], bkb[C::TM], bke[C::TM];
  __shared__ int slow_rows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 2u * C::NPT);
      mbar_init(&empty[s], unsigned(C::NCW));
    }
  }
  __syncthreads();

  if (warp < C::NPW) {
    // ------------------------------------------------------------------ producers
    const int tid = threadIdx.x;
    int stage = 0;
    unsigned phase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const GTile tl = tiles[t];
      // the previous tile's copies were all issued: the row tables can be rewritten
      asm volatile("bar.sync 1, %0;\n" ::"n"(C::NPT));
      if (tid == 0) slow_rows = 0;
      __syncwarp();
      if (warp == 0) {
        // segments -> rows: a warp-wide scan of the segments' row counts
        int base = 0;
        for (int s0 = tl.seg_begin; s0 < tl.seg_end && base < C::TM; s0 += 32) {
          GSeg sg;
          sg.rows = 0;
          if (s0 + lane < tl.seg_end) sg = segs[s0 + lane];
          int incl = sg.rows;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
          }
          const int start = base + incl - sg.rows;
          if (sg.rows > 0) {
            const bool pad = sg.ke <= sg.kb;  // zero rows (alignment padding)
            const double* p0 = pad ? nullptr : bufs.p[sg.buf] + sg.off - sg.kb;
            const bool full_range = sg.kb == 0 && sg.ke == tl.klen && (sg.ld & 1) == 0 &&
                                    (reinterpret_cast<uintptr_t>(p0) & 15) == 0;
            if (!pad && !full_range) slow_rows = 1;
            for (int x = 0; x < sg.rows && start + x < C::TM; ++x) {
              akb[start + x] = pad ? 0 : sg.kb;
              ake[start + x] = pad ? 0 : sg.ke;
              arow[start + x] = pad ? nullptr : p0 + int64_t(x) * sg.ld;
            }
          }
          base += __shfl_sync(0xffffffffu, incl, 31);
        }
      } else {
        const double* B = bufs.p[tl.b_buf] + tl.b_off;
        for (int j = lane; j < C::TM; j += 32) {
          brow[j] = B + int64_t(j) * tl.b_ld;
          bkb[j] = 0;
          bke[j] = tl.klen;
        }
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(C::NPT));
      const double* safe = bufs.p[tl.b_buf] + tl.b_off;
      const bool a_fast = slow_rows == 0;
      const bool b_fast = (tl.b_ld & 1) == 0 && (reinterpret_cast<uintptr_t>(safe) & 15) == 0;
      const int rows8 = (tl.rows + 7) & ~7, cols8 = (tl.cols + 7) & ~7;
      const int nch = max(1, (tl.klen + C::KC - 1) / C::KC);
      for (int c = 0; c < nch; ++c) {
        mbar_wait(&empty[stage], phase ^ 1u);
        double* sP = smem + stage * C::STAGE;
        const unsigned sp = static_cast<unsigned>(__cvta_generic_to_shared(sP));
        const unsigned sq = static_cast<unsigned>(__cvta_generic_to_shared(sP + C::OPSZ));
        const int kk0 = c * C::KC;
        const bool inside = kk0 + C::KC <= tl.klen;
        gws_stage<C>(sp, arow, akb, ake, safe, tl.rows, rows8, kk0, a_fast && inside, tid);
        gws_stage<C>(sq, brow, bkb, bke, safe, tl.cols, cols8, kk0, b_fast && inside, tid);
        if (tid == 0) {
          desc[stage].used = max(0, min(C::KC, tl.klen - kk0));
          desc[stage].last = c + 1 == nch;
        }
        mbar_cp_async_arrive(&full[stage]);
        mbar_arrive(&full[stage]);
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------------- consumers
  const int cw = warp - C::NPW;
  int stage = 0;
  unsigned phase = 0;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const GTile tl = tiles[t];
    const int nfc = (tl.cols + 7) >> 3;
    unsigned amask = 0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
      if (cw * 16 + a * 8 < tl.rows) amask |= 1u << a;
    double acc[2][8][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 8; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    while (true) {
      mbar_wait(&full[stage], phase);
      const GwsDesc d = desc[stage];
      const double* sP = smem + stage * C::STAGE;
      const double* sQ = sP + C::OPSZ;
      if (d.used > 0 && amask) {
        switch (nfc) {
          case 1: gws_mma<C, 1>(acc, sP, sQ, d.used, cw, lane, amask); break;
          case 2: gws_mma<C, 2>(acc, sP, sQ, d.used, cw, lane, amask); break;
          case 3: gws_mma<C, 3>(acc, sP, sQ, d.used, cw, lane, amask); break;
          case 4: gws_mma<C, 4>(acc, sP, sQ, d.used, cw, lane, amask); break;
          case 5: gws_mma<C, 5>(acc, sP, sQ, d.used, cw, lane, amask); break;
          case 6: gws_mma<C, 6>(acc, sP, sQ, d.used, cw, lane, amask); break;
          case 7: gws_mma<C, 7>(acc, sP, sQ, d.used, cw, lane, amask); break;
          default: gws_mma<C, 8>(acc, sP, sQ, d.used, cw, lane, amask); break;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == C::STAGES) {
        stage = 0;
        phase ^= 1u;
      }
      if (d.last) break;
    }
    double* out = bufs.p[tl.out_buf] + tl.out_off;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int r = cw * 16 + a * 8 + (lane >> 2);
#pragma unroll
      for (int b = 0; b < 8; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cc = b * 8 + (lane & 3) * 2 + h;
          if (r < tl.rows && cc < tl.cols) out[r + int64_t(cc) * tl.out_ld] = acc[a][b][h];
        }
    }
  }
}

}  // namespace hx

// Warp-specialized, persistent version of the grouped sum-of-products GEMM (gemm.cuh).
//
// Same work lists (Tile / Group / Term, hx_types.h), same staging layouts, same DMMA inner
// loop and epilogue modes; what changes is who does what and how they synchronize.
// Profiles of the classic kernel (profiles/r02_form_kernel_ncu.txt) show the term-formation
// launches issue ~12 instructions per DMMA: every thread of the CTA walks the tile's term
// cursor and computes the staging addresses of every segment, between two CTA barriers per
// chunk, with 4 warps per scheduler -- the tensor pipe idles while all warps of a CTA are
// in the integer part.  Here:
//   * NPW producer warps walk the cursor, issue the cp.async staging of a STAGES-deep
//     ring of chunks and publish each chunk's descriptor (slots used, layouts, fragment
//     masks, last-of-tile flag);
//   * 4 consumer warps (2 x 2, 32 x 32 each, as before) only read fragments from shared
//     memory and issue DMMA, then run the tile's epilogue;
//   * the ring is synchronized by mbarriers: full[s] completes when every producer
//     thread's copies have landed (cp.async.mbarrier.arrive.noinc) and its plain shared
//     stores are released (mbarrier.arrive); empty[s] when the 4 consumer warps are done
//     with the stage.  No CTA-wide barrier in the main loop;
//   * CTAs are persistent (grid = resident CTAs, tiles round-robin), so the producers
//     stage the next tile's first chunks while the consumers finish a tile and write it
//     out: short-K tiles (term formation, ~70 slots) no longer pay a pipeline fill each.
#pragma once
#include <cstdint>

#include "gemm.cuh"

namespace hx {

template <int KC_, int STAGES_, int NPW_, int MINB_>
struct WsCfg {
  static constexpr int TM = 64;
  static constexpr int KC = KC_;
  static constexpr int STAGES = STAGES_;
  static constexpr int NPW = NPW_;                 // producer warps
  static constexpr int NCW = 4;                    // consumer warps (2 x 2)
  static constexpr int NPT = 32 * NPW;             // producer threads
  static constexpr int THREADS = 32 * (NPW + NCW);
  static constexpr int MINB = MINB_;
  static constexpr int LDI = TM + 4;
  static constexpr int LDK = KC + 4;
  static constexpr int OPSZ = (KC * LDI > TM * LDK) ? KC * LDI : TM * LDK;
  static constexpr int WT = TM / 2;
  static constexpr int FR = WT / 8;
  static constexpr int STAGE = 2 * OPSZ;           // P + Q (doubles)
  static constexpr int MAXSEG = 8;
  static constexpr int SMEM = STAGES * STAGE * 8;  // + static: barriers, descriptors
};

// short-K batches (term formation): 16-slot chunks, 3 stages (60 KB), 3 CTAs per SM
using Ws64s = WsCfg<16, 3, 2, 3>;
// long-K batches (materialization, sketches): 32-slot chunks, 3 stages, 2 CTAs per SM
using Ws64 = WsCfg<32, 3, 2, 2>;

struct WsDesc {
  int32_t used;    // slots filled (0: empty tile)
  int32_t tile;    // tile index (consumers' epilogue)
  uint8_t akc, bkc, last, pad;
  uint8_t amask[2], bmask[2];  // per consumer row half (wm) / column half (wn)
};

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(a)
               : "memory");
}
__device__ __forceinline__ void mbar_cp_async_arrive(uint64_t* bar) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

// Producer cursor over the tile's (group, term, k offset), reading the term and group
// records through warp-wide windows: lane i holds record base + i (one coalesced load per
// window), the current one is broadcast by shuffles.  The cursor of the classic kernel
// loads each record when it reaches it, a chain of dependent L2 round trips per segment
// that bounds how fast the producers can stage (term formation: ~4 segments per chunk).
struct WsCursor {
  int g, g_end, t, t_end, k0;
  int tbase, tn;  // term window [tbase, tbase + tn)
  int gbase, gn;  // group window
  Term tm;        // current term (uniform over the warp)
  Term wt;        // this lane's term of the window
  Group wg;       // this lane's group of the window
};

__device__ __forceinline__ Term shfl_term(const Term& x, int src) {
  static_assert(sizeof(Term) == 48, "Term layout");
  Term y;
  const int* xi = reinterpret_cast<const int*>(&x);
  int* yi = reinterpret_cast<int*>(&y);
#pragma unroll
  for (int w = 0; w < 12; ++w) yi[w] = __shfl_sync(0xffffffffu, xi[w], src);
  return y;
}

__device__ __forceinline__ bool ws_next_term(WsCursor& c, const Group* __restrict__ groups,
                                             const Term* __restrict__ terms, int lane) {
  while (true) {
    ++c.t;
    if (c.t < c.t_end) {
      if (c.t < c.tbase || c.t >= c.tbase + c.tn) {
        c.tbase = c.t;
        c.tn = min(32, c.t_end - c.t);
        if (lane < c.tn) c.wt = terms[c.t + lane];
      }
      c.tm = shfl_term(c.wt, c.t - c.tbase);
      c.k0 = 0;
      if (c.tm.k > 0) return true;
      continue;
    }
    ++c.g;
    if (c.g >= c.g_end) return false;
    if (c.g >= c.gbase + c.gn) {
      c.gbase = c.g;
      c.gn = min(32, c.g_end - c.g);
      if (lane < c.gn) c.wg = groups[c.g + lane];
    }
    const int src = c.g - c.gbase;
    c.t = __shfl_sync(0xffffffffu, c.wg.t_begin, src) - 1;
    c.t_end = __shfl_sync(0xffffffffu, c.wg.t_end, src);
  }
}

__device__ __forceinline__ void ws_cursor_init(WsCursor& c, const Tile& tl) {
  c.g = tl.g_begin - 1;
  c.g_end = tl.g_end;
  c.t = c.t_end = 0;
  c.k0 = 0;
  c.tbase = c.tn = 0;
  c.gbase = c.gn = 0;
}

// Producer-side staging of n slots of one operand segment (layouts as stage_seg in
// gemm.cuh), spread over the C::NPT producer threads (tid in [0, NPT)).
template <class C>
__device__ __forceinline__ void ws_stage_seg(unsigned sbase, const double* base,
                                             const double* safe, int ld, int kc, int lo,
                                             int hi, int slot0, int n, int tid, int ilo = 0,
                                             int ihi = C::TM) {
  // rows outside [ilo, ihi) are left as they are: the caller guarantees that no consumer
  // reads them (a chunk made of this one segment, whose fragment mask excludes them)
  constexpr int TM = C::TM;
  if (kc == 0) {
    const bool al = ((reinterpret_cast<uintptr_t>(base) & 15) == 0) && ((ld & 1) == 0) &&
                    (((lo | hi) & 1) == 0);
    if (al) {
      constexpr int PR = TM / 2, CL = C::NPT / PR;
      const int p = tid % PR, c = tid / PR;
      const int i = 2 * p;
      if (i < ilo || i >= ihi) return;
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
      constexpr int CL = C::NPT / TM;
      const int i = tid % TM, c = tid / TM;
      if (i < ilo || i >= ihi) return;
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
      constexpr int PK = C::KC / 2, RL = C::NPT / PK;
      const int q = tid % PK, r = tid / PK;
      const int kk = 2 * q;
      if (kk < n) {
        const bool pair = kk + 1 < n;
        const int i0 = r + (ilo > r ? (ilo - r + RL - 1) / RL * RL : 0);
        const double* src = base + kk + int64_t(i0) * ld;
        unsigned dst = sbase + 8u * unsigned(i0 * C::LDK + slot0 + kk);
        for (int i = i0; i < ihi; i += RL) {
          const bool v = i >= lo && i < hi;
          if (pair) cp_async16(dst, v ? src : safe, v ? 16 : 0);
          else cp_async8(dst, v ? src : safe, v ? 8 : 0);
          src += int64_t(RL) * ld;
          dst += 8u * RL * C::LDK;
        }
      }
    } else {
      constexpr int RL = C::NPT / C::KC;
      const int kk = tid % C::KC, r = tid / C::KC;
      if (kk < n) {
        const int i0 = r + (ilo > r ? (ilo - r + RL - 1) / RL * RL : 0);
        const double* src = base + kk + int64_t(i0) * ld;
        unsigned dst = sbase + 8u * unsigned(i0 * C::LDK + slot0 + kk);
        for (int i = i0; i < ihi; i += RL) {
          const bool v = i >= lo && i < hi;
          cp_async8(dst, v ? src : safe, v ? 8 : 0);
          src += int64_t(RL) * ld;
          dst += 8u * RL * C::LDK;
        }
      }
    }
  }
}

template <class C>
__device__ __forceinline__ void ws_stage_cols(unsigned sbase, const double* const* colp,
                                              int64_t off, const double* safe, int lo, int hi,
                                              int slot0, int n, int tid, bool aligned) {
  constexpr int PK = C::KC / 2, RL = C::NPT / PK;
  const int q = tid % PK, r = tid / PK;
  const int kk = 2 * q;
  if (kk >= n) return;
  const bool pair = kk + 1 < n;
  if (aligned && ((off | slot0) & 1) == 0) {
    // every column pointer of the tile is 16-byte aligned (flag set with the table): one
    // 16-byte copy per slot pair and row, no per-row alignment test
    unsigned dst = sbase + 8u * unsigned(r * C::LDK + slot0 + kk);
#pragma unroll 4
    for (int i = r; i < C::TM; i += RL) {
      const bool v = i >= lo && i < hi;
      const double* src = v ? colp[i] + off + kk : safe;
      if (pair) cp_async16(dst, src, v ? 16 : 0);
      else cp_async8(dst, src, v ? 8 : 0);
      dst += 8u * RL * C::LDK;
    }
    return;
  }
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

template <class C>
__device__ __forceinline__ void ws_zero_slots(double* s, int kc, int a, int b, int tid) {
  const int n = b - a;
  if (n <= 0) return;
  for (int e = tid; e < n * C::TM; e += C::NPT) {
    const int kk = a + e / C::TM, i = e % C::TM;
    s[kc ? i * C::LDK + kk : kk * C::LDI + i] = 0.0;
  }
}

// 8-row fragments of tile half w (rows [w WT, w WT + WT)) that meet [lo, hi): bit a set
// when fragment a does (the consumers skip the others).
template <class C>
__device__ __forceinline__ unsigned ws_frag_mask(int lo, int hi, int w) {
  const int l = max(lo - w * C::WT, 0), h = min(hi - w * C::WT, C::WT);
  if (h <= l) return 0u;
  return (2u << ((h - 1) >> 3)) - (1u << (l >> 3));
}

// Producer: fill one stage from the cursor; returns the descriptor (all producer threads
// compute it identically).
template <class C, bool GC>
__device__ __forceinline__ WsDesc ws_build_chunk(double* sP, double* sQ, WsCursor& cur,
                                                 bool& have, const Group* __restrict__ groups,
                                                 const Term* __restrict__ terms,
                                                 const BufPtrs& bufs, const Tile& tl,
                                                 const double* const* colp, int tid,
                                                 bool colp_aligned) {
  WsDesc d;
  d.used = 0;
  d.amask[0] = d.amask[1] = d.bmask[0] = d.bmask[1] = 0;
  d.akc = cur.tm.a_kc;
  d.bkc = cur.tm.b_kc ? 1 : 0;
  d.last = 0;
  d.pad = 0;
  const unsigned sp = static_cast<unsigned>(__cvta_generic_to_shared(sP));
  const unsigned sq = static_cast<unsigned>(__cvta_generic_to_shared(sQ));
  int nseg = 0;
  while (have && d.used < C::KC && nseg < C::MAXSEG) {
    const Term& tm = cur.tm;
    if (tm.a_kc != d.akc || (tm.b_kc ? 1 : 0) != d.bkc) break;
    const int n = min(C::KC - d.used, tm.k - cur.k0);
    const int i0 = tl.row0 - tm.r_lo, j0 = tl.col0 - tm.c_lo;
    const int rlo = max(0, -i0), rhi = min(int(tl.rows), tm.rows - i0);
    const int clo = max(0, -j0), chi = min(int(tl.cols), tm.cols - j0);
    const double* A = bufs.p[tm.a_buf] + tm.a_off;
    const double* B = bufs.p[tm.b_buf] + tm.b_off;
    const double* pa =
        tm.a_kc ? A + cur.k0 + int64_t(i0) * tm.a_ld : A + i0 + int64_t(cur.k0) * tm.a_ld;
    const double* pb =
        tm.b_kc ? B + cur.k0 + int64_t(j0) * tm.b_ld : B + j0 + int64_t(cur.k0) * tm.b_ld;
    // a segment that fills the chunk on its own (the stacked cores: K = a cluster size)
    // stages only the row fragments it covers; the consumers' masks skip the others
    int ilo = 0, ihi = C::TM;
    if (n == C::KC) {
      ilo = rhi > rlo ? (rlo & ~7) : 0;
      ihi = rhi > rlo ? min((rhi + 7) & ~7, C::TM) : 0;
    }
    ws_stage_seg<C>(sp, pa, A, tm.a_ld, tm.a_kc, rlo, rhi, d.used, n, tid, ilo, ihi);
    if (GC && tm.b_kc == 2)
      ws_stage_cols<C>(sq, colp, tm.b_off + cur.k0, bufs.p[BUF_A], clo, chi, d.used, n, tid,
                       colp_aligned);
    else
      ws_stage_seg<C>(sq, pb, B, tm.b_ld, tm.b_kc, clo, chi, d.used, n, tid);
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      d.amask[w] |= uint8_t(ws_frag_mask<C>(rlo, rhi, w));
      d.bmask[w] |= uint8_t(ws_frag_mask<C>(clo, chi, w));
    }
    d.used += n;
    ++nseg;
    cur.k0 += n;
    if (cur.k0 >= tm.k) have = ws_next_term(cur, groups, terms, tid & 31);
  }
  const int padded = (d.used + 3) & ~3;
  ws_zero_slots<C>(sP, d.akc, d.used, padded, tid);
  ws_zero_slots<C>(sQ, d.bkc, d.used, padded, tid);
  return d;
}

template <class C, int AK, int BK>
__device__ __forceinline__ void ws_mma_t(double (&acc)[C::FR][C::FR][2], const double* sP,
                                         const double* sQ, int used, int wm, int wn,
                                         int lane, unsigned amask) {
  constexpr int SA_I = AK ? C::LDK : 1, SA_K = AK ? 1 : C::LDI;
  constexpr int SB_I = BK ? C::LDK : 1, SB_K = BK ? 1 : C::LDI;
  const int ksteps = (used + 3) >> 2;
  const int r = lane >> 2, q = lane & 3;
  const double* pa = sP + (wm * C::WT + r) * SA_I + q * SA_K;
  const double* pb = sQ + (wn * C::WT + r) * SB_I + q * SB_K;
  if (amask != (1u << C::FR) - 1) {
    // partially covered row half (stacked cores: a leaf's k_l rows, 8-row aligned): only
    // the covered 8-row fragments, row-fragment-outer so that the skip is one warp-uniform
    // branch per fragment and chunk (B fragments re-read from shared memory per row)
#pragma unroll
    for (int a = 0; a < C::FR; ++a) {
      if (!((amask >> a) & 1u)) continue;
      for (int ks = 0; ks < ksteps; ++ks) {
        const double af = pa[a * 8 * SA_I + ks * 4 * SA_K];
        double bf[C::FR];
#pragma unroll
        for (int b = 0; b < C::FR; ++b) bf[b] = pb[b * 8 * SB_I + ks * 4 * SB_K];
#pragma unroll
        for (int b = 0; b < C::FR; ++b) dmma_8x8x4(acc[a][b][0], acc[a][b][1], af, bf[b]);
      }
    }
    return;
  }
  // column fragments outside every segment multiply staged zeros (unconditional DMMA)
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
}

// GC: the launch has MODE_GCOL tiles (term formation); launches without a column-record
// table (materialization, sketches) compile the column-pointer path out.
template <class C, bool GC>
__global__ void __launch_bounds__(C::THREADS, C::MINB) grouped_gemm_ws_kernel(
    const Tile* __restrict__ tiles, const Group* __restrict__ groups,
    const Term* __restrict__ terms, const __grid_constant__ BufPtrs bufs,
    double* __restrict__ sumsq, int n_tiles, const ColRec* __restrict__ gcols) {
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t full[C::STAGES], empty[C::STAGES];
  __shared__ WsDesc desc[C::STAGES];
  __shared__ const double* colp[C::TM];
  __shared__ unsigned colp_bad[C::NPW];
  __shared__ double red[C::NCW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      // every producer thread arrives twice per fill: once when its copies land, once
      // (release) after its plain shared stores
      mbar_init(&full[s], 2u * C::NPT);
      mbar_init(&empty[s], unsigned(C::NCW));
    }
  }
  __syncthreads();

  if (warp < C::NPW) {
    // ------------------------------------------------------------------ producers
    const int tid = threadIdx.x;  // [0, NPT)
    int stage = 0;
    unsigned phase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const Tile tl = tiles[t];
      bool colp_aligned = false;
      if (GC && tl.mode == MODE_GCOL) {
        // the previous tile's copies were all issued (they captured their source pointers),
        // so the table can be rewritten once every producer is past them
        asm volatile("bar.sync 1, %0;\n" ::"n"(C::NPT));
        bool bad = false;
        if (tid < tl.cols) {
          const int j = tl.col0 + tid;
          int idx = tl.aux;
          ColRec r = gcols[idx];
          while (j >= r.col + r.k) r = gcols[++idx];
          const double* p = bufs.p[r.buf] + r.src_off + int64_t(j - r.col) * r.ld;
          colp[tid] = p;
          bad = (reinterpret_cast<uintptr_t>(p) & 15) != 0;
        }
        const unsigned anybad = __ballot_sync(0xffffffffu, bad);
        if ((tid & 31) == 0) colp_bad[tid >> 5] = anybad;
        asm volatile("bar.sync 1, %0;\n" ::"n"(C::NPT));
        unsigned allbad = 0;
#pragma unroll
        for (int w = 0; w < C::NPW; ++w) allbad |= colp_bad[w];
        colp_aligned = allbad == 0;
      }
      WsCursor cur;
      ws_cursor_init(cur, tl);
      bool have = ws_next_term(cur, groups, terms, tid & 31);
      do {
        mbar_wait(&empty[stage], phase ^ 1u);
        double* sP = smem + stage * C::STAGE;
        WsDesc d = ws_build_chunk<C, GC>(sP, sP + C::OPSZ, cur, have, groups, terms, bufs, tl,
                                     colp, tid, colp_aligned);
        d.tile = t;
        d.last = have ? 0 : 1;
        if (tid == 0) desc[stage] = d;
        mbar_cp_async_arrive(&full[stage]);
        mbar_arrive(&full[stage]);
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      } while (have);
    }
    return;
  }

  // -------------------------------------------------------------------- consumers
  const int cw = warp - C::NPW;
  const int wm = cw >> 1, wn = cw & 1;
  int stage = 0;
  unsigned phase = 0;
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    double acc[C::FR][C::FR][2];
#pragma unroll
    for (int a = 0; a < C::FR; ++a)
#pragma unroll
      for (int b = 0; b < C::FR; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    while (true) {
      mbar_wait(&full[stage], phase);
      const WsDesc d = desc[stage];
      const double* sP = smem + stage * C::STAGE;
      if (d.used > 0 && d.amask[wm] && d.bmask[wn]) {
        const unsigned am = d.amask[wm];
        switch (d.akc * 2 + d.bkc) {
          case 0: ws_mma_t<C, 0, 0>(acc, sP, sP + C::OPSZ, d.used, wm, wn, lane, am); break;
          case 1: ws_mma_t<C, 0, 1>(acc, sP, sP + C::OPSZ, d.used, wm, wn, lane, am); break;
          case 2: ws_mma_t<C, 1, 0>(acc, sP, sP + C::OPSZ, d.used, wm, wn, lane, am); break;
          default: ws_mma_t<C, 1, 1>(acc, sP, sP + C::OPSZ, d.used, wm, wn, lane, am); break;
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
    // epilogue.  Plain stores (term formation, materialization) take a branch-free path:
    // short-K tiles spend a third of the consumers' time here otherwise.
    const Tile tl = tiles[t];
    double* out = bufs.p[tl.out_buf] + tl.out_off;
    double ss = 0.0;
    if (tl.mode != MODE_ADD && tl.mode != MODE_RESID_SUMSQ) {
      const int r0 = wm * C::WT + (lane >> 2), c0 = wn * C::WT + (lane & 3) * 2;
      double* base = out + r0 + int64_t(c0) * tl.out_ld;
      const bool sq = tl.mode == MODE_STORE_SUMSQ;
      const bool full = tl.rows == C::TM && tl.cols == C::TM;
      if (full) {
#pragma unroll
        for (int b = 0; b < C::FR; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double* p = base + int64_t(b * 8 + h) * tl.out_ld;
#pragma unroll
            for (int a = 0; a < C::FR; ++a) p[a * 8] = acc[a][b][h];
          }
      } else {
        const int nr = tl.rows - r0, nc = tl.cols - c0;  // this lane's rows a * 8 < nr
#pragma unroll
        for (int b = 0; b < C::FR; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double* p = base + int64_t(b * 8 + h) * tl.out_ld;
            const bool cok = b * 8 + h < nc;
#pragma unroll
            for (int a = 0; a < C::FR; ++a)
              if (cok && a * 8 < nr) {
                p[a * 8] = acc[a][b][h];
                ss += acc[a][b][h] * acc[a][b][h];
              }
          }
      }
      if (sq && full) {
#pragma unroll
        for (int a = 0; a < C::FR; ++a)
#pragma unroll
          for (int b = 0; b < C::FR; ++b) ss += acc[a][b][0] * acc[a][b][0] + acc[a][b][1] * acc[a][b][1];
      }
    } else {
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
                v = *dst - v;
              } else {
                if (tl.mode == MODE_ADD) v += *dst;
                *dst = v;
              }
              ss += v * v;
            }
          }
        }
      }
    }
    if (tl.mode == MODE_STORE_SUMSQ || tl.mode == MODE_RESID_SUMSQ) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) red[cw] = ss;
      asm volatile("bar.sync 2, %0;\n" ::"n"(32 * C::NCW));
      if (cw == 0 && lane == 0) {
        double s = 0.0;
        for (int w = 0; w < C::NCW; ++w) s += red[w];
        sumsq[tl.aux] = s;
      }
      asm volatile("bar.sync 2, %0;\n" ::"n"(32 * C::NCW));
    }
  }
}

}  // namespace hx

// Row-parallel Householder QR (LAPACK dgeqr2 + dorg2r semantics) of the many tall, thin
// panels of the recompression (Y = T Omega, B^T = T^T Q; p up to a few thousand rows,
// q = sketch width).
//
// Every thread owns the rows i = t, t + nt, ... of the panel.  A reflector step needs
// w_c = v^T M[:, c] for all trailing columns c: each thread accumulates its rows' share for
// 32 columns at a time in registers, one 31-shuffle transpose-reduction per warp sums them
// (lane x ends up with column x), and the CTA variant adds the per-warp sums through shared
// memory.  The update M[i, c] -= tau w_c v_i is then again row-parallel.  Compared with one
// column per lane/warp (serial length-p dot products) this keeps all threads busy and
// replaces q^2 reductions by q^2/32 transpose-reductions per panel.
//
//   qr_rows_warp_kernel  one warp per panel, panel in its shared-memory slice
//   qr_rows_cta_kernel   one CTA (256-1024 threads) per panel, in shared memory when it fits,
//                        else in place in HBM (coalesced: consecutive threads, consecutive rows)
#pragma once
#include <cstdint>

#include "dense_la.cuh"

namespace hx {

// Sum over the 32 lanes of part[0..31]; afterwards lane l returns the total of part[l].
__device__ __forceinline__ double transpose_reduce32(double (&part)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int x = 0; x < o; ++x) {
      const double send = up ? part[x] : part[x + o];
      const double keep = up ? part[x + o] : part[x];
      part[x] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return part[0];
}

template <bool CTA>
__device__ __forceinline__ void grp_sync() {
  if (CTA)
    __syncthreads();
  else
    __syncwarp();
}

// Apply H_j = I - tau v v^T, v = (1, M[j+1:p, j]), to columns j+1..q-1 (rows j..p-1).
// wsum: 32 doubles shared by the group; red: 32 per warp (CTA only).
template <bool CTA>
__device__ void rows_apply(double* M, int ld, int p, int q, int j, double tau, double* wsum,
                           double* red, int t, int nt) {
  const double* v = M + int64_t(j) * ld;
  const int lane = t & 31, warp = t >> 5;
  for (int c0 = j + 1; c0 < q; c0 += 32) {
    const int nc = min(32, q - c0);
    double part[32];
#pragma unroll
    for (int x = 0; x < 32; ++x) part[x] = 0.0;
    for (int i = j + 1 + t; i < p; i += nt) {
      const double vi = v[i];
      const double* row = M + i + int64_t(c0) * ld;
#pragma unroll
      for (int x = 0; x < 32; ++x)
        if (x < nc) part[x] = fma(vi, row[int64_t(x) * ld], part[x]);
    }
    const double w = transpose_reduce32(part, lane);
    if (CTA) {
      red[warp * 32 + lane] = w;
      __syncthreads();
      if (t < 32) {
        double s = 0.0;
        for (int k = 0; k < (nt >> 5); ++k) s += red[k * 32 + t];
        if (t < nc) wsum[t] = tau * (s + M[j + int64_t(c0 + t) * ld]);
      }
      __syncthreads();
    } else {
      if (lane < nc) wsum[lane] = tau * (w + M[j + int64_t(c0 + lane) * ld]);
      __syncwarp();
    }
    if (t < nc) M[j + int64_t(c0 + t) * ld] -= wsum[t];
    for (int i = j + 1 + t; i < p; i += nt) {
      const double vi = v[i];
      double* row = M + i + int64_t(c0) * ld;
#pragma unroll
      for (int x = 0; x < 32; ++x)
        if (x < nc) row[int64_t(x) * ld] = fma(-wsum[x], vi, row[int64_t(x) * ld]);
    }
    grp_sync<CTA>();
  }
}

// In-place QR of M (p x q, ld): R (q x q, ld ldr) to Rout, M overwritten by the explicit Q.
// tau_s: q doubles, wsum: 32, red: 32 per warp (CTA).
template <bool CTA>
__device__ void rows_householder_qr(double* M, int ld, int p, int q, double* Rout, int ldr,
                                    double* tau_s, double* wsum, double* red) {
  const int t = CTA ? int(threadIdx.x) : int(threadIdx.x & 31);
  const int nt = CTA ? int(blockDim.x) : 32;
  for (int j = 0; j < q; ++j) {
    double* x = M + int64_t(j) * ld;
    double part = 0.0;
    for (int i = j + 1 + t; i < p; i += nt) part = fma(x[i], x[i], part);
    const double xn2 = CTA ? block_sum(part, red) : warp_sum(part);
    const double alpha = j < p ? x[j] : 0.0;
    double tau, beta;
    if (xn2 == 0.0) {
      tau = 0.0;
      beta = alpha;
    } else {
      beta = -copysign(hypot(alpha, sqrt(xn2)), alpha);
      tau = (beta - alpha) / beta;
      const double scal = 1.0 / (alpha - beta);
      for (int i = j + 1 + t; i < p; i += nt) x[i] *= scal;
    }
    grp_sync<CTA>();
    if (t == 0) {
      if (j < p) x[j] = beta;
      tau_s[j] = tau;
    }
    if (tau != 0.0) rows_apply<CTA>(M, ld, p, q, j, tau, wsum, red, t, nt);
    grp_sync<CTA>();
  }
  for (int e = t; e < q * q; e += nt) {
    const int i = e % q, c = e / q;
    Rout[i + int64_t(c) * ldr] = (i <= c && i < p) ? M[i + int64_t(c) * ld] : 0.0;
  }
  grp_sync<CTA>();
  for (int j = q - 1; j >= 0; --j) {
    const double tau = tau_s[j];
    if (j < q - 1 && tau != 0.0) rows_apply<CTA>(M, ld, p, q, j, tau, wsum, red, t, nt);
    double* x = M + int64_t(j) * ld;
    for (int i = j + 1 + t; i < p; i += nt) x[i] *= -tau;
    for (int i = t; i < j && i < p; i += nt) x[i] = 0.0;
    if (t == 0 && j < p) x[j] = 1.0 - tau;
    grp_sync<CTA>();
  }
}

// One warp per panel; slice = p * q + q + 32 doubles per warp.
__global__ void qr_rows_warp_kernel(const QrJob* __restrict__ jobs, int n_jobs, int slice) {
  extern __shared__ __align__(16) double dsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int jid = blockIdx.x * (blockDim.x >> 5) + warp;
  if (jid >= n_jobs) return;
  const QrJob jb = jobs[jid];
  const int p = jb.p, q = jb.q;
  double* M = dsm + int64_t(warp) * slice;
  double* tau_s = M + int64_t(p) * q;
  double* wsum = tau_s + q;
  const int64_t n = int64_t(p) * q;
  const int64_t lx = jb.lx();
  for (int64_t e = lane; e < n; e += 32) M[e] = jb.X[e % p + (e / p) * lx];
  __syncwarp();
  rows_householder_qr<false>(M, p, p, q, jb.R, jb.lr(), tau_s, wsum, nullptr);
  for (int64_t e = lane; e < n; e += 32) jb.X[e % p + (e / p) * lx] = M[e];
}

// One CTA of NT threads per panel; use_smem: stage the panel (p * q doubles) in dynamic
// shared memory.  Taller panels get more threads (one or two rows each).
template <int NT>
__global__ void __launch_bounds__(NT, (NT <= 256 ? 2 : 1))
    qr_rows_cta_kernel(const QrJob* __restrict__ jobs, int use_smem) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ double tau_s[JAC_QMAX];
  __shared__ double wsum[32];
  __shared__ double red[NT];
  const QrJob jb = jobs[blockIdx.x];
  const int p = jb.p, q = jb.q;
  const int64_t n = int64_t(p) * q;
  const int64_t lx = jb.lx();
  if (use_smem) {
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) dsm[e] = jb.X[e % p + (e / p) * lx];
    __syncthreads();
    rows_householder_qr<true>(dsm, p, p, q, jb.R, jb.lr(), tau_s, wsum, red);
    __syncthreads();
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) jb.X[e % p + (e / p) * lx] = dsm[e];
  } else {
    rows_householder_qr<true>(jb.X, int(lx), p, q, jb.R, jb.lr(), tau_s, wsum, red);
  }
}

// ---------------------------------------------------------------------------------------
// Register-resident variant for the bulk of the panels (p <= 32 NW RPT, q <= QM <= 32): one
// CTA of NW warps per panel, every thread holds RPT full rows of the panel in registers, so
// a reflector step costs RPT QM FMAs for the partial dots, QM/16 transpose-reductions and
// RPT QM FMAs for the update -- no shared-memory traffic for the panel itself.

// Sum over the 32 lanes of part[0..N-1] (N = 16 or 32); lane l returns column l % N.
template <int N>
__device__ __forceinline__ double transpose_reduce(double (&part)[N], int lane) {
#pragma unroll
  for (int o = N / 2; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int x = 0; x < o; ++x) {
      const double send = up ? part[x] : part[x + o];
      const double keep = up ? part[x + o] : part[x];
      part[x] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  double v = part[0];
#pragma unroll
  for (int o = N; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int QM>
__device__ __forceinline__ double reg_pick(const double (&row)[QM], int j) {
  double v = 0.0;
#pragma unroll
  for (int x = 0; x < QM; ++x) v = (x == j) ? row[x] : v;
  return v;
}

template <int NW, int QM, int RPT>
__global__ void __launch_bounds__(NW * 32, NW == 1 ? 8 : 16 / NW) qr_reg_kernel(const QrJob* __restrict__ jobs) {
  constexpr int NT = NW * 32;
  __shared__ double red[NW][QM];
  __shared__ double wsum[QM];
  __shared__ double taus[QM];
  __shared__ double bc;
  const QrJob jb = jobs[blockIdx.x];
  const int p = jb.p, q = jb.q;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int ii[RPT];
  double a[RPT][QM];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    ii[r] = t + r * NT;
#pragma unroll
    for (int x = 0; x < QM; ++x)
      a[r][x] = (x < q && ii[r] < p) ? jb.X[ii[r] + int64_t(x) * jb.lx()] : 0.0;
  }
  // group sum of a scalar
  auto gsum = [&](double v) {
    v = warp_sum(v);
    if (NW == 1) return v;
    if (lane == 0) red[warp][0] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w][0];
    __syncthreads();
    return s;
  };
  // wsum[x] = sum over rows of v_i a[i][x] (visible to every thread on return)
  auto gdots = [&](const double (&v)[RPT]) {
#pragma unroll
    for (int h = 0; h < QM / 16; ++h) {
      double part[16];
#pragma unroll
      for (int x = 0; x < 16; ++x) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < RPT; ++r) s = fma(v[r], a[r][h * 16 + x], s);
        part[x] = s;
      }
      const double w = transpose_reduce<16>(part, lane);
      if (lane < 16) red[warp][h * 16 + lane] = w;
    }
    __syncthreads();
    if (t < QM) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < NW; ++k) s += red[k][t];
      wsum[t] = s;
    }
    __syncthreads();
  };
  // a[i][x] -= tau wsum[x] v_i for x > j
  auto gupdate = [&](const double (&v)[RPT], int j, double tau) {
#pragma unroll
    for (int x = 0; x < QM; ++x)
      if (x > j) {
        const double w = tau * wsum[x];
#pragma unroll
        for (int r = 0; r < RPT; ++r) a[r][x] = fma(-w, v[r], a[r][x]);
      }
    __syncthreads();
  };
  auto setcol = [&](int j, const double (&n)[RPT]) {
#pragma unroll
    for (int x = 0; x < QM; ++x)
      if (x == j) {
#pragma unroll
        for (int r = 0; r < RPT; ++r) a[r][x] = n[r];
      }
  };
  for (int j = 0; j < q; ++j) {
    double xs[RPT];
    double part = 0.0;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      xs[r] = reg_pick<QM>(a[r], j);
      if (ii[r] > j) part = fma(xs[r], xs[r], part);
      if (ii[r] == j) bc = xs[r];
    }
    const double xn2 = gsum(part);
    __syncthreads();
    const double alpha = bc;
    double tau = 0.0, beta = alpha;
    if (xn2 != 0.0) {
      beta = -copysign(hypot(alpha, sqrt(xn2)), alpha);
      tau = (beta - alpha) / beta;
      const double scal = 1.0 / (alpha - beta);
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        if (ii[r] > j) xs[r] *= scal;
    }
    // column j := beta on the diagonal, v below, R above (unchanged)
    double n[RPT], v[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      n[r] = ii[r] == j ? beta : xs[r];
      v[r] = ii[r] > j ? xs[r] : (ii[r] == j ? 1.0 : 0.0);
    }
    setcol(j, n);
    if (t == 0) taus[j] = tau;
    if (tau != 0.0) {
      gdots(v);
      gupdate(v, j, tau);
    } else {
      __syncthreads();
    }
  }
  // R (q x q): the upper triangle of rows 0..q-1
#pragma unroll
  for (int r = 0; r < RPT; ++r)
    if (ii[r] < q) {
#pragma unroll
      for (int x = 0; x < QM; ++x)
        if (x < q) jb.R[ii[r] + int64_t(x) * jb.lr()] = (ii[r] <= x) ? a[r][x] : 0.0;
    }
  // explicit Q (dorg2r)
  for (int j = q - 1; j >= 0; --j) {
    const double tau = taus[j];
    double v[RPT], n[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const double xr = reg_pick<QM>(a[r], j);
      v[r] = ii[r] > j ? xr : (ii[r] == j ? 1.0 : 0.0);
      n[r] = ii[r] > j ? -tau * xr : (ii[r] == j ? 1.0 - tau : 0.0);
    }
    if (j < q - 1 && tau != 0.0) {
      gdots(v);
      gupdate(v, j, tau);
    }
    setcol(j, n);
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r)
    if (ii[r] < p) {
#pragma unroll
      for (int x = 0; x < QM; ++x)
        if (x < q) jb.X[ii[r] + int64_t(x) * jb.lx()] = a[r][x];
    }
}

}  // namespace hx

namespace hx {

// ---------------------------------------------------------------------------------------
// TSQR of tall panels (p > 256 rows, q <= 64): the panel is cut into row blocks of
// 128..255 rows, each block is factored in place by the kernels above (explicit Q_i,
// R_i stacked into S), S is factored the same way until one block remains, and the
// explicit Q is assembled top-down: every block's Q_i is multiplied in place by its q x q
// slice of the explicit Q of the level above.  One CTA per 64-row slab of a block.
struct TsMul {
  double* X;         // slab (rows x q, ld ldx), overwritten by X * Qs
  const double* Qs;  // q x q slice (ld ldq)
  int ldx, ldq, rows, q;
};

constexpr int TS_SLAB = 64;
constexpr int TS_QMAX = 64;

__global__ void __launch_bounds__(256) tsqr_apply_kernel(const TsMul* __restrict__ jobs) {
  extern __shared__ __align__(16) double tsm[];
  double* xs = tsm;                      // TS_SLAB x q, ld TS_SLAB
  double* qs = tsm + TS_SLAB * TS_QMAX;  // q x q, ld TS_QMAX
  const TsMul jb = jobs[blockIdx.x];
  const int rows = jb.rows, q = jb.q;
  for (int e = threadIdx.x; e < TS_SLAB * q; e += blockDim.x) {
    const int i = e & (TS_SLAB - 1), c = e / TS_SLAB;
    xs[e] = i < rows ? jb.X[i + int64_t(c) * jb.ldx] : 0.0;
  }
  for (int e = threadIdx.x; e < q * q; e += blockDim.x) {
    const int i = e % q, c = e / q;
    qs[i + c * TS_QMAX] = jb.Qs[i + int64_t(c) * jb.ldq];
  }
  __syncthreads();
  const int i = threadIdx.x & (TS_SLAB - 1);
  for (int c = threadIdx.x / TS_SLAB; c < q; c += blockDim.x / TS_SLAB) {
    double acc = 0.0;
    for (int k = 0; k < q; ++k) acc = fma(xs[i + k * TS_SLAB], qs[k + c * TS_QMAX], acc);
    if (i < rows) jb.X[i + int64_t(c) * jb.ldx] = acc;
  }
}

}  // namespace hx

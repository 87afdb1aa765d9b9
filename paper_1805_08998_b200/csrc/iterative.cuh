// Matrix-free compressors of the far output blocks on the implicit sum (the `aca`,
// `bilanczos` and `randomized` tags of compress, compressors.py:441-452).
//
// Each far block's operator S = T + sum_t P_t Q_t is either a materialized tile (T only,
// the block formed by the grouped GEMM) or, for the implicit route, its terms clipped to
// the block (factor pairs and dense x dense pairs: P_t rows x k, Q_t k x cols) plus the
// materialized sub-block part T_sub.  A *team* -- one warp for small blocks, one CTA for
// large or implicit ones -- runs the reference's iteration for one block, touching S only
// through the LinearMap accesses the reference uses (compressors.py:34-67):
//   row(i) / col(j)          ACA's residual rows and columns (LinearMap.row/col :53-61,
//                            SumExpression.apply_transpose/apply sumexpr.py:59-75)
//   apply(x) / apply_t(w)    Lanczos and randomized matvecs
// On the implicit route a row is sum_t P_t(i, :) Q_t (a k-vector gathered from P_t, then
// a coalesced sweep over Q_t), a matvec first reduces Q_t x over the team's warps (one dot
// per term column) and then sweeps P_t.  Team-wide reductions are warp shuffles (plus one
// shared-memory pass for CTA teams); control flow is uniform over the team.
//
// The algorithms restate the reference line by line (thresholds, two-hit stop, pivoting,
// breakdown restarts, per-block seeds); the exact SVD recompressions that follow them
// (ACA's truncate(eps/2), the Lanczos core SVD) run on the batched QR / Jacobi / select
// kernels of the sketch route (runtime.cu).
#pragma once
#include <cfloat>
#include <climits>
#include <cstdint>

#include "dense_la.cuh"
#include "np_random.cuh"

namespace hx {

enum IterTag : int32_t { ITER_ACA = 0, ITER_GKL = 1, ITER_RAND = 2 };

// One term of an implicit block, clipped to it: covers block rows [ri, ri + rn) and
// columns [ci, ci + cn); P(ii, kk) = P[ii * ps + kk * pk] (ii = row - ri),
// Q(kk, jj) = Q[jj * qs + kk * qk] (jj = col - ci).
struct IterTerm {
  const double* P;
  const double* Q;
  int64_t ps, pk, qs, qk;
  int32_t k, ri, rn, ci, cn;
  int32_t koff;  // first of this term's k entries in the job's tz scratch
};

struct IterJob {
  const double* T;  // materialized tile / T_sub (column-major m x n, ld ldT) or nullptr
  int64_t ldT;
  int32_t m, n;
  int32_t t_begin, t_end;  // IterTerm range
  int32_t kcap;            // columns of L / U / Wb
  int32_t node;            // block id (per-block seed)
  double* L;    // m x kcap  ACA crosses l / Lanczos left basis / randomized basis
  double* U;    // n x kcap  ACA crosses u / Lanczos rows^T / randomized rows / Omega
  double* Wb;   // n x kcap  Lanczos right basis (nullptr otherwise)
  double* vm;   // 2 m scratch
  double* vn;   // 3 n scratch
  double* tz;   // scratch: sum of term ranks (matvec dots) + 2 kcap + 8
  uint8_t* used;  // m + n flags (ACA)
};

struct IterOut {
  int32_t k;        // columns produced
  int32_t degraded; // ACA ran out of rows without a certified zero
  int32_t capped;   // kcap too small: rerun with more columns
  int32_t matvecs;  // CountingMap total (compressors.py:88-119)
};

struct IterParams {
  int32_t tag;     // IterTag
  int32_t policy;  // 0 EpsRank, 1 FixedRank
  double eps;
  int32_t k_max;
  int32_t q;       // randomized subspace iterations (CompressorKind.q)
  uint64_t seed;   // CompressorKind.seed
};

// ---------------------------------------------------------------- teams
template <int NW>
struct Team {  // NW warps = the whole CTA
  static constexpr int size = NW * 32;
  int rank;
  double* red;  // >= 2 * NW doubles of shared memory
  int* redi;    // >= NW ints
  __device__ Team(double* r, int* ri) : rank(threadIdx.x), red(r), redi(ri) {}
  __device__ int warp() const { return rank >> 5; }
  __device__ void sync() const { __syncthreads(); }
  __device__ double sum(double v) const {
    v = warp_sum(v);
    __syncthreads();
    if ((rank & 31) == 0) red[rank >> 5] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w];
    return s;
  }
  __device__ void sum2(double& a, double& b) const {
    a = warp_sum(a);
    b = warp_sum(b);
    __syncthreads();
    if ((rank & 31) == 0) {
      red[rank >> 5] = a;
      red[NW + (rank >> 5)] = b;
    }
    __syncthreads();
    a = 0.0;
    b = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      a += red[w];
      b += red[NW + w];
    }
  }
  // max of v over the team, ties to the smaller index (numpy argmax: first occurrence)
  __device__ void argmax(double& v, int& idx) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov > v || (ov == v && oi < idx)) {
        v = ov;
        idx = oi;
      }
    }
    __syncthreads();
    if ((rank & 31) == 0) {
      red[rank >> 5] = v;
      redi[rank >> 5] = idx;
    }
    __syncthreads();
    v = red[0];
    idx = redi[0];
    for (int w = 1; w < NW; ++w)
      if (red[w] > v || (red[w] == v && redi[w] < idx)) {
        v = red[w];
        idx = redi[w];
      }
  }
  __device__ int imin(int x) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = min(x, __shfl_xor_sync(0xffffffffu, x, o));
    __syncthreads();
    if ((rank & 31) == 0) redi[rank >> 5] = x;
    __syncthreads();
    int r = redi[0];
    for (int w = 1; w < NW; ++w) r = min(r, redi[w]);
    return r;
  }
};

template <>
struct Team<1> {  // one warp of a multi-warp CTA
  static constexpr int size = 32;
  int rank;
  __device__ Team(double*, int*) : rank(threadIdx.x & 31) {}
  __device__ int warp() const { return 0; }
  __device__ void sync() const { __syncwarp(); }
  __device__ double sum(double v) const { return warp_sum(v); }
  __device__ void sum2(double& a, double& b) const {
    a = warp_sum(a);
    b = warp_sum(b);
  }
  __device__ void argmax(double& v, int& idx) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov > v || (ov == v && oi < idx)) {
        v = ov;
        idx = oi;
      }
    }
  }
  __device__ int imin(int x) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = min(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
  }
};

// out[c] = sum_{i < len} X[i + c * ldx] * y[i] for c < K (one warp per dot), then sync.
template <int NW>
__device__ void team_dots(const Team<NW>& tm, const double* X, int64_t ldx, int K,
                          const double* y, int len, double* out) {
  tm.sync();
  const int lane = tm.rank & 31;
  for (int c = tm.warp(); c < K; c += NW) {
    const double* x = X + int64_t(c) * ldx;
    double acc = 0.0;
    for (int i = lane; i < len; i += 32) acc += x[i] * y[i];
    acc = warp_sum(acc);
    if (lane == 0) out[c] = acc;
  }
  tm.sync();
}

// v -= X[:, :K] (X[:, :K]^T v), twice (_reorth, compressors.py:264-268); v owned by rows.
template <int NW>
__device__ void team_reorth(const Team<NW>& tm, const double* X, int64_t ldx, int K, double* v,
                            int len, double* coef) {
  if (K <= 0) return;
  for (int pass = 0; pass < 2; ++pass) {
    team_dots(tm, X, ldx, K, v, len, coef);
    for (int i = tm.rank; i < len; i += Team<NW>::size) {
      double acc = 0.0;
      for (int c = 0; c < K; ++c) acc += X[i + int64_t(c) * ldx] * coef[c];
      v[i] -= acc;
    }
  }
}

template <int NW>
__device__ double team_norm(const Team<NW>& tm, const double* v, int len) {
  double s = 0.0;
  for (int i = tm.rank; i < len; i += Team<NW>::size) s += v[i] * v[i];
  return sqrt(tm.sum(s));
}

// ---------------------------------------------------------------- the block operator
struct IterOp {
  const double* T;
  int64_t ldT;
  int m, n;
  const IterTerm* tb;
  int nt;
  double* tz;

  // first index >= lo owned by the thread (indices owned by rank mod size)
  template <int S>
  __device__ static int first_owned(int rank, int lo) {
    return lo + (((rank - lo) % S) + S) % S;
  }

  // out[j] = S[i, j] (the residual-free row; rows are owned by column index)
  template <int NW>
  __device__ void row(const Team<NW>& tm, int i, double* out) const {
    constexpr int S = Team<NW>::size;
    for (int j = tm.rank; j < n; j += S) out[j] = T ? T[i + int64_t(j) * ldT] : 0.0;
    for (int t = 0; t < nt; ++t) {
      const IterTerm x = tb[t];
      if (i < x.ri || i >= x.ri + x.rn) continue;
      const double* p = x.P + int64_t(i - x.ri) * x.ps;
      for (int j = first_owned<S>(tm.rank, x.ci); j < x.ci + x.cn; j += S) {
        const double* q = x.Q + int64_t(j - x.ci) * x.qs;
        double acc = 0.0;
        for (int kk = 0; kk < x.k; ++kk) acc += p[kk * x.pk] * q[kk * x.qk];
        out[j] += acc;
      }
    }
  }
  template <int NW>
  __device__ void col(const Team<NW>& tm, int j, double* out) const {
    constexpr int S = Team<NW>::size;
    for (int i = tm.rank; i < m; i += S) out[i] = T ? T[i + int64_t(j) * ldT] : 0.0;
    for (int t = 0; t < nt; ++t) {
      const IterTerm x = tb[t];
      if (j < x.ci || j >= x.ci + x.cn) continue;
      const double* q = x.Q + int64_t(j - x.ci) * x.qs;
      for (int i = first_owned<S>(tm.rank, x.ri); i < x.ri + x.rn; i += S) {
        const double* p = x.P + int64_t(i - x.ri) * x.ps;
        double acc = 0.0;
        for (int kk = 0; kk < x.k; ++kk) acc += p[kk * x.pk] * q[kk * x.qk];
        out[i] += acc;
      }
    }
  }
  // y = S x (x: n, y: m, rows owned); x must be complete (synced) on entry
  template <int NW>
  __device__ void apply(const Team<NW>& tm, const double* x, double* y) const {
    constexpr int S = Team<NW>::size;
    tm.sync();
    if (nt) {
      const int lane = tm.rank & 31;
      int pair = 0;
      for (int t = 0; t < nt; ++t) {
        const IterTerm e = tb[t];
        for (int kk = 0; kk < e.k; ++kk, ++pair) {
          if (pair % NW != tm.warp()) continue;
          double acc = 0.0;
          for (int jj = lane; jj < e.cn; jj += 32)
            acc += e.Q[int64_t(jj) * e.qs + int64_t(kk) * e.qk] * x[e.ci + jj];
          acc = warp_sum(acc);
          if (lane == 0) tz[e.koff + kk] = acc;
        }
      }
      tm.sync();
    }
    for (int i = tm.rank; i < m; i += S) {
      double acc = 0.0;
      if (T)
        for (int j = 0; j < n; ++j) acc += T[i + int64_t(j) * ldT] * x[j];
      for (int t = 0; t < nt; ++t) {
        const IterTerm e = tb[t];
        if (i < e.ri || i >= e.ri + e.rn) continue;
        const double* p = e.P + int64_t(i - e.ri) * e.ps;
        for (int kk = 0; kk < e.k; ++kk) acc += p[kk * e.pk] * tz[e.koff + kk];
      }
      y[i] = acc;
    }
  }
  // z = S^T w (w: m, z: n, columns owned); w complete on entry
  template <int NW>
  __device__ void apply_t(const Team<NW>& tm, const double* w, double* z) const {
    constexpr int S = Team<NW>::size;
    tm.sync();
    if (nt) {
      const int lane = tm.rank & 31;
      int pair = 0;
      for (int t = 0; t < nt; ++t) {
        const IterTerm e = tb[t];
        for (int kk = 0; kk < e.k; ++kk, ++pair) {
          if (pair % NW != tm.warp()) continue;
          double acc = 0.0;
          for (int ii = lane; ii < e.rn; ii += 32)
            acc += e.P[int64_t(ii) * e.ps + int64_t(kk) * e.pk] * w[e.ri + ii];
          acc = warp_sum(acc);
          if (lane == 0) tz[e.koff + kk] = acc;
        }
      }
      tm.sync();
    }
    for (int j = tm.rank; j < n; j += S) {
      double acc = 0.0;
      if (T) {
        const double* col = T + int64_t(j) * ldT;
        for (int i = 0; i < m; ++i) acc += col[i] * w[i];
      }
      for (int t = 0; t < nt; ++t) {
        const IterTerm e = tb[t];
        if (j < e.ci || j >= e.ci + e.cn) continue;
        const double* q = e.Q + int64_t(j - e.ci) * e.qs;
        for (int kk = 0; kk < e.k; ++kk) acc += q[kk * e.qk] * tz[e.koff + kk];
      }
      z[j] = acc;
    }
  }
};

// ---------------------------------------------------------------- ACA (compressors.py:162-247)
template <int NW>
__device__ void iter_aca(const Team<NW>& tm, const IterOp& op, const IterJob& jb,
                         const IterParams& prm, IterOut& out) {
  constexpr int S = Team<NW>::size;
  const int m = jb.m, n = jb.n, mu = min(m, n);
  const bool eps_mode = prm.policy == 0;
  const int kstop = eps_mode ? mu : min(prm.k_max, mu);
  uint8_t* used_r = jb.used;
  uint8_t* used_c = jb.used + m;
  double* row = jb.vn;
  double* col = jb.vm;
  double* L = jb.L;
  double* U = jb.U;
  for (int e = tm.rank; e < m + n; e += S) jb.used[e] = 0;
  tm.sync();
  double norm_sq = 0.0;
  int i = 0, k = 0, rows_zero = 0, hits = 0, deg = 0, mv = 0, capped = 0;
  while (k < kstop) {
    if (k >= jb.kcap) {
      capped = 1;
      break;
    }
    if (i < 0 || used_r[i]) {
      int f = INT_MAX;
      for (int e = tm.rank; e < m; e += S)
        if (!used_r[e]) {
          f = e;
          break;
        }
      f = tm.imin(f);
      if (f == INT_MAX) {  // rows exhausted: certified zero only if every row sampled zero
        deg = (k == 0 && rows_zero == m) ? 0 : 1;
        break;
      }
      i = f;
    }
    tm.sync();
    if (tm.rank == 0) used_r[i] = 1;
    op.row(tm, i, row);
    ++mv;
    // residual row u_hat = row(i) - sum_c u_c l_c[i]; column pivot over unused columns
    double best = -1.0;
    int bj = INT_MAX;
    for (int j = tm.rank; j < n; j += S) {
      double uh = row[j];
      for (int c = 0; c < k; ++c) uh -= U[j + int64_t(c) * n] * L[i + int64_t(c) * m];
      row[j] = uh;
      const double a = used_c[j] ? 0.0 : fabs(uh);
      if (a > best) {
        best = a;
        bj = j;
      }
    }
    tm.argmax(best, bj);
    tm.sync();
    const double scale = sqrt(norm_sq);
    if (best <= 1e-14 * scale || best == 0.0) {  // residual row carries no signal
      if (k > 0) break;
      ++rows_zero;
      i = -1;
      continue;
    }
    const double pivot = row[bj];
    double nu2 = 0.0;
    for (int j = tm.rank; j < n; j += S) {
      const double u = row[j] / pivot;
      U[j + int64_t(k) * n] = u;
      nu2 += u * u;
    }
    op.col(tm, bj, col);
    ++mv;
    double nl2 = 0.0;
    for (int r = tm.rank; r < m; r += S) {
      double l = col[r];
      for (int c = 0; c < k; ++c) l -= L[r + int64_t(c) * m] * U[bj + int64_t(c) * n];
      L[r + int64_t(k) * m] = l;
      nl2 += l * l;
    }
    tm.sum2(nl2, nu2);
    const double update = sqrt(nl2) * sqrt(nu2);
    if (update <= 1e-15 * scale || update == 0.0) break;  // cross adds nothing
    if (eps_mode) {
      const double acc = k ? scale : update;
      hits = (update <= prm.eps * acc) ? hits + 1 : 0;
    }
    double cross = 0.0;
    if (k) {  // incremental ||L U||_F^2 in cross space
      team_dots(tm, L, m, k, L + int64_t(k) * m, m, jb.tz);
      team_dots(tm, U, n, k, U + int64_t(k) * n, n, jb.tz + k);
      for (int c = 0; c < k; ++c) cross += jb.tz[c] * jb.tz[k + c];
    }
    tm.sync();
    if (tm.rank == 0) used_c[bj] = 1;
    norm_sq += 2.0 * cross + update * update;
    ++k;
    if (hits >= 2) break;
    // next pivot row: largest |l| over unused rows
    best = -1.0;
    int bi = INT_MAX;
    for (int r = tm.rank; r < m; r += S) {
      const double a = used_r[r] ? 0.0 : fabs(L[r + int64_t(k - 1) * m]);
      if (a > best) {
        best = a;
        bi = r;
      }
    }
    tm.argmax(best, bi);
    i = best > 0.0 ? bi : -1;
    tm.sync();
  }
  out.k = k;
  out.degraded = deg;
  out.capped = capped;
  out.matvecs = mv;
}

// -------------------------------------------- Golub-Kahan-Lanczos (compressors.py:271-365)
template <int NW>
__device__ void draw_normals(const Team<NW>& tm, NpRng& g, double* v, int n) {
  tm.sync();
  if (tm.rank == 0)
    for (int e = 0; e < n; ++e) v[e] = g.normal();
  tm.sync();
}

template <int NW>
__device__ void iter_gkl(const Team<NW>& tm, const IterOp& op, const IterJob& jb,
                         const IterParams& prm, IterOut& out) {
  constexpr int S = Team<NW>::size;
  const int m = jb.m, n = jb.n, mu = min(m, n);
  const bool eps_mode = prm.policy == 0;
  const int kstop = eps_mode ? mu : min(prm.k_max, mu);
  NpRng g;
  if (tm.rank == 0) {
    uint64_t lo, hi;
    block_seed(prm.seed, jb.node, lo, hi);
    g.seed(lo, hi);
  }
  double* w = jb.vn;
  double* wn = jb.vn + n;
  double* q = jb.vm;
  double* coef = jb.tz;
  draw_normals(tm, g, w, n);
  {
    const double nw = team_norm(tm, w, n);
    for (int j = tm.rank; j < n; j += S) w[j] /= nw;
  }
  double beta_prev = 0.0, norm_sq = 0.0;
  int k = 0, probes = 0, hits = 0, mv = 0, capped = 0;
  while (k < kstop) {
    if (k >= jb.kcap) {
      capped = 1;
      break;
    }
    op.apply(tm, w, q);
    ++mv;
    if (k > 0 && beta_prev != 0.0)
      for (int i = tm.rank; i < m; i += S) q[i] -= beta_prev * jb.L[i + int64_t(k - 1) * m];
    team_reorth(tm, jb.L, m, k, q, m, coef);
    const double alpha = team_norm(tm, q, m);
    if (alpha <= 1e-14 * fmax(sqrt(norm_sq), 1e-300)) {
      // breakdown: a fresh direction orthogonal to span(W)
      if (probes >= 3 || k >= n) break;
      ++probes;
      draw_normals(tm, g, w, n);
      team_reorth(tm, jb.Wb, n, k, w, n, coef);
      const double nw = team_norm(tm, w, n);
      if (nw == 0.0) break;
      for (int j = tm.rank; j < n; j += S) w[j] /= nw;
      beta_prev = 0.0;
      continue;
    }
    if (eps_mode && k > 0) {
      const double upd = hypot(alpha, beta_prev);
      hits = (upd <= prm.eps * sqrt(fmax(norm_sq, 0.0))) ? hits + 1 : 0;
    }
    for (int i = tm.rank; i < m; i += S) jb.L[i + int64_t(k) * m] = q[i] / alpha;
    for (int j = tm.rank; j < n; j += S) jb.Wb[j + int64_t(k) * n] = w[j];
    probes = 0;
    tm.sync();
    op.apply_t(tm, jb.L + int64_t(k) * m, wn);
    ++mv;
    for (int j = tm.rank; j < n; j += S) wn[j] -= alpha * w[j];
    team_reorth(tm, jb.Wb, n, k + 1, wn, n, coef);
    const double beta = team_norm(tm, wn, n);
    norm_sq += alpha * alpha + beta * beta;
    if (beta <= 1e-14 * sqrt(norm_sq)) {  // invariant subspace, no tail coupling
      for (int j = tm.rank; j < n; j += S) jb.U[j + int64_t(k) * n] = alpha * w[j];
      ++k;
      break;
    }
    for (int j = tm.rank; j < n; j += S) {
      wn[j] /= beta;
      jb.U[j + int64_t(k) * n] = alpha * w[j] + beta * wn[j];
    }
    ++k;
    if (hits >= 2) break;
    beta_prev = beta;
    double* t = w;
    w = wn;
    wn = t;
    tm.sync();
  }
  tm.sync();
  out.k = k;
  out.degraded = 0;
  out.capped = capped;
  out.matvecs = mv;
}

// ---------------------------- randomized range finders (compressors.py:368-428)
template <int NW>
__device__ void iter_rand_adaptive(const Team<NW>& tm, const IterOp& op, const IterJob& jb,
                                   const IterParams& prm, IterOut& out) {
  constexpr int S = Team<NW>::size;
  const int m = jb.m, n = jb.n, mu = min(m, n);
  NpRng g;
  if (tm.rank == 0) {
    uint64_t lo, hi;
    block_seed(prm.seed, jb.node, lo, hi);
    g.seed(lo, hi);
  }
  double* omega = jb.vn;
  double* l = jb.vm;
  double norm_sq = 0.0;
  int k = 0, hits = 0, mv = 0, capped = 0;
  for (int it = 0; it < mu; ++it) {
    if (k >= jb.kcap) {
      capped = 1;
      break;
    }
    draw_normals(tm, g, omega, n);
    op.apply(tm, omega, l);
    ++mv;
    const double l0 = team_norm(tm, l, m);
    team_reorth(tm, jb.L, m, k, l, m, jb.tz);
    const double ln = team_norm(tm, l, m);
    if (ln <= 1e-14 * fmax(sqrt(norm_sq), l0)) break;  // image already captured
    double* lh = jb.L + int64_t(k) * m;
    for (int i = tm.rank; i < m; i += S) lh[i] = l[i] / ln;
    tm.sync();
    double* u = jb.U + int64_t(k) * n;
    op.apply_t(tm, lh, u);
    ++mv;
    double uu = 0.0, ll = 0.0;
    for (int j = tm.rank; j < n; j += S) uu += u[j] * u[j];
    for (int i = tm.rank; i < m; i += S) ll += lh[i] * lh[i];
    tm.sum2(uu, ll);
    norm_sq += uu;
    ++k;
    if (k > 1 && sqrt(ll) * sqrt(uu) <= prm.eps * sqrt(norm_sq)) {
      if (++hits >= 2) break;
    } else {
      hits = 0;
    }
  }
  tm.sync();
  out.k = k;
  out.degraded = 0;
  out.capped = capped;
  out.matvecs = mv;
}

// orthonormal columns of X[:, :K] (ld ldx) by CGS2, column by column (np.linalg.qr's Q up
// to column signs; the products Q Q^T S the caller forms do not see the signs)
template <int NW>
__device__ void team_orth(const Team<NW>& tm, double* X, int64_t ldx, int K, int len,
                          double* coef) {
  constexpr int S = Team<NW>::size;
  for (int c = 0; c < K; ++c) {
    double* x = X + int64_t(c) * ldx;
    const double n0 = team_norm(tm, x, len);
    team_reorth(tm, X, ldx, c, x, len, coef);
    const double nx = team_norm(tm, x, len);
    const double inv = (nx > 1e-14 * n0 && nx > 0.0) ? 1.0 / nx : 0.0;
    for (int i = tm.rank; i < len; i += S) x[i] *= inv;
    tm.sync();
  }
}

template <int NW>
__device__ void iter_rand_fixed(const Team<NW>& tm, const IterOp& op, const IterJob& jb,
                                const IterParams& prm, IterOut& out) {
  const int m = jb.m, n = jb.n;
  const int kk = min(prm.k_max, min(m, n));
  if (kk > jb.kcap) {
    tm.sync();
    out.k = 0;
    out.degraded = 0;
    out.capped = 1;
    out.matvecs = 0;
    return;
  }
  // Omega = standard_normal((n, kk)), drawn in C order, stored column-major in U
  tm.sync();
  if (tm.rank == 0) {
    NpRng g;
    uint64_t lo, hi;
    block_seed(prm.seed, jb.node, lo, hi);
    g.seed(lo, hi);
    for (int64_t e = 0; e < int64_t(n) * kk; ++e)
      jb.U[(e / kk) + (e % kk) * int64_t(n)] = g.normal();
  }
  tm.sync();
  int mv = 0;
  for (int c = 0; c < kk; ++c) op.apply(tm, jb.U + int64_t(c) * n, jb.L + int64_t(c) * m);
  mv += kk;
  team_orth(tm, jb.L, m, kk, m, jb.tz);
  for (int it = 0; it < prm.q; ++it) {
    for (int c = 0; c < kk; ++c) op.apply_t(tm, jb.L + int64_t(c) * m, jb.U + int64_t(c) * n);
    team_orth(tm, jb.U, n, kk, n, jb.tz);
    for (int c = 0; c < kk; ++c) op.apply(tm, jb.U + int64_t(c) * n, jb.L + int64_t(c) * m);
    team_orth(tm, jb.L, m, kk, m, jb.tz);
    mv += 2 * kk;
  }
  for (int c = 0; c < kk; ++c) op.apply_t(tm, jb.L + int64_t(c) * m, jb.U + int64_t(c) * n);
  mv += kk;
  tm.sync();
  out.k = kk;
  out.degraded = 0;
  out.capped = 0;
  out.matvecs = mv;
}

// One team per job: NW == 1 packs 4 independent warps per CTA (small blocks), NW > 1 is a
// CTA per job (large or implicit blocks).
template <int NW>
__global__ void __launch_bounds__(NW == 1 ? 128 : NW * 32)
    iter_kernel(const IterJob* __restrict__ jobs, const IterTerm* __restrict__ terms,
                IterOut* __restrict__ outs, int n_jobs, IterParams prm) {
  __shared__ double red[2 * (NW == 1 ? 1 : NW)];
  __shared__ int redi[NW == 1 ? 1 : NW];
  const int job = NW == 1 ? int(blockIdx.x) * 4 + int(threadIdx.x >> 5) : int(blockIdx.x);
  if (job >= n_jobs) return;
  const Team<NW> tm(red, redi);
  const IterJob jb = jobs[job];
  IterOp op{jb.T, jb.ldT, jb.m, jb.n, terms + jb.t_begin, jb.t_end - jb.t_begin, jb.tz};
  // tz: term dots first, then the k-vectors of the iterations
  int ksum = 0;
  if (op.nt) {
    const IterTerm& last = op.tb[op.nt - 1];
    ksum = last.koff + last.k;
  }
  IterJob j2 = jb;
  j2.tz = jb.tz + ((ksum + 7) & ~7);
  IterOut o{0, 0, 0, 0};
  if (prm.tag == ITER_ACA)
    iter_aca(tm, op, j2, prm, o);
  else if (prm.tag == ITER_GKL)
    iter_gkl(tm, op, j2, prm, o);
  else if (prm.policy == 1)
    iter_rand_fixed(tm, op, j2, prm, o);
  else
    iter_rand_adaptive(tm, op, j2, prm, o);
  if (tm.rank == 0) outs[job] = o;
}

// out (n x k) = U (n x k) R^T for the upper-triangular k x k R: the right factor of ACA's
// truncation, (L U^T)^T Q_L = U R_L^T (lowrank.py:93-104); grid (job, row chunks of 128).
struct UrJob {
  const double* U;
  const double* R;
  double* out;
  int n, k;
};

__global__ void __launch_bounds__(128) ur_product_kernel(const UrJob* __restrict__ jobs) {
  const UrJob jb = jobs[blockIdx.x];
  for (int j = blockIdx.y * 128 + threadIdx.x; j < jb.n; j += 128 * gridDim.y) {
    for (int c = 0; c < jb.k; ++c) {
      double acc = 0.0;
      for (int kk = c; kk < jb.k; ++kk)
        acc += jb.U[j + int64_t(kk) * jb.n] * jb.R[c + int64_t(kk) * jb.k];
      jb.out[j + int64_t(c) * jb.n] = acc;
    }
  }
}

// numpy standard normals of one seeded stream (diagnostics / parity tests)
__global__ void np_normals_kernel(uint64_t lo, uint64_t hi, double* out, int64_t n) {
  if (threadIdx.x || blockIdx.x) return;
  NpRng g;
  g.seed(lo, hi);
  for (int64_t e = 0; e < n; ++e) out[e] = g.normal();
}

}  // namespace hx

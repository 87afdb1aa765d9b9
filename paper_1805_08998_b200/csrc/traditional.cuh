// Traditional-mode far leaves: hmult_traditional (/root/reference/pkg/src/hmat/multiply.py:
// 140-263) on the device.
//
// The planner (plan.cpp, trad_leaf / trad_pair) turns every far leaf into a tree of values:
//   items  a term of the product's term list on its own block -- a thin product formed by
//          the term-formation GEMMs (TN_LR), or a dense x dense pair kept as the factor pair
//          (D_A rows, D_B columns) of rank |rho| (TN_DD);
//   folds  fast_truncate_sum (lowrank.py:123-138) of their children: acc = T(c0 + c1),
//          acc = T(acc + c_i), ... with T = truncate (lowrank.py:107-113); a fold over one
//          dense item is from_dense (lowrank.py:50-54); the leaf root sorts its children by
//          decreasing norm first (multiply.py:222-224);
//   stacks one truncation of all children side by side (the best approximation of a pair
//          product: the "dense-svd" converter, compressors.py:431-438).
// Children sit on sub-blocks of their parent (the zero padding of _pad_child,
// multiply.py:103-109, becomes a row / column offset of the gathered factors).
//
// Execution is a data-flow sweep in waves: every fold whose children are all known
// advances one truncation per wave, so a wave is one batch of independent truncations
//   gather [acc | child] into panels L (m x K), R (n x K)       trad_gather_kernel
//   Householder QR of the panels that are taller than K         run_qr
//   core C = R_L R_R^T (<= K x K)                               grouped DMMA GEMM
//   one-sided Jacobi SVD of C, select_rank                      run_jacobi, select_rank_kernel
//   factors (Q_L W_r S_r, Q_R V_r) written where they are used  small_product_kernel
// after which the host reads the ranks (one small copy per wave) and places the outputs:
// intermediate sums in a ping-pong arena, finished values in per-wave keep buffers.
#pragma once

namespace hx {

struct TVal {  // low-rank value L R^T on a node's block (L m x k, R n x k)
  const double* L = nullptr;
  const double* R = nullptr;
  int64_t ldl = 0, ldr = 0;
  int8_t lrow = 0, rrow = 0;  // 1: row-major factor, element (i, kk) at i * ld + kk
  int k = 0;
  double norm = 0.0;
};

// One factor of one input, copied into rows [row0, row0 + rows) of a panel column range
// (every other row of those columns is zeroed: the padding of a child block).
struct TSeg {
  const double* src;
  double* dst;
  int64_t lds;
  int ldd, row0, rows, total, k, rowmajor;
};

__global__ void __launch_bounds__(256) trad_gather_kernel(const TSeg* __restrict__ segs) {
  const TSeg s = segs[blockIdx.x];
  const int64_t ne = int64_t(s.total) * s.k;
  for (int64_t e = threadIdx.x + int64_t(blockIdx.y) * blockDim.x; e < ne;
       e += int64_t(blockDim.x) * gridDim.y) {
    const int i = int(e % s.total), kk = int(e / s.total);
    const int r = i - s.row0;
    double v = 0.0;
    if (r >= 0 && r < s.rows)
      v = s.rowmajor ? s.src[kk + int64_t(r) * s.lds] : s.src[r + int64_t(kk) * s.lds];
    s.dst[i + int64_t(kk) * s.ldd] = v;
  }
}

// ||L R^T||_F = sqrt(sum_ab (L^T L)_ab (R^T R)_ab), LowRank.norm's Gram trick
// (lowrank.py:38-43); 32 x 32 tiles of the two Gram matrices (upper triangle of tiles).
struct TNormJob {
  const double* L;
  const double* R;
  int64_t ldl, ldr;
  int m, n, k, lrow, rrow;
  double* out;
};

__global__ void __launch_bounds__(256) trad_norm_kernel(const TNormJob* __restrict__ jobs) {
  __shared__ double sa[32][33], sb[32][33];
  __shared__ double red[8];
  const TNormJob jb = jobs[blockIdx.x];
  const int k = jb.k, nt = (k + 31) / 32, tid = threadIdx.x, ta = tid & 31;
  double total = 0.0;
  for (int t0 = 0; t0 < nt; ++t0)
    for (int t1 = t0; t1 < nt; ++t1) {
      double g[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
      for (int side = 0; side < 2; ++side) {
        const double* F = side ? jb.R : jb.L;
        const int64_t ld = side ? jb.ldr : jb.ldl;
        const int rowm = side ? jb.rrow : jb.lrow;
        const int rows = side ? jb.n : jb.m;
        for (int r0 = 0; r0 < rows; r0 += 32) {
          __syncthreads();
          for (int e = tid; e < 1024; e += 256) {
            const int rr = e & 31, cc = e >> 5, r = r0 + rr;
            const int a = t0 * 32 + cc, b = t1 * 32 + cc;
            sa[rr][cc] = (r < rows && a < k) ? (rowm ? F[a + r * ld] : F[r + a * ld]) : 0.0;
            sb[rr][cc] = (r < rows && b < k) ? (rowm ? F[b + r * ld] : F[r + b * ld]) : 0.0;
          }
          __syncthreads();
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int tb = (tid >> 5) + 8 * e;
            double acc = 0.0;
#pragma unroll 8
            for (int rr = 0; rr < 32; ++rr) acc += sa[rr][ta] * sb[rr][tb];
            g[side][e] += acc;
          }
        }
      }
      double part = 0.0;
#pragma unroll
      for (int e = 0; e < 4; ++e) part += g[0][e] * g[1][e];
      total += (t0 == t1 ? 1.0 : 2.0) * part;
    }
  const double s = block_sum(total, red);
  if (tid == 0) *jb.out = sqrt(fmax(s, 0.0));
}

// norm of a truncated value: sqrt(sum_{i < rank} sigma_i^2)
__global__ void trad_sig_norm_kernel(const double* const* __restrict__ sig,
                                     const int* __restrict__ rank, double* __restrict__ out,
                                     int n) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double s = 0.0;
  for (int i = 0; i < rank[j]; ++i) s += sig[j][i] * sig[j][i];
  out[j] = sqrt(s);
}

}  // namespace hx


// Warp-level dense linear algebra for the many small far blocks (sketch width <= 32).
//
// The CTA kernels of dense_la.cuh spend most of their time in __syncthreads between the
// q column steps of a QR and the q-1 rounds of every Jacobi sweep.  For small blocks one
// warp owns one block and synchronises only with __syncwarp:
//   warp_jacobi_kernel  one-sided Jacobi SVD of a q x q factor, one column per lane held in
//                       registers, partner columns exchanged with shuffles (q <= QM)
#pragma once
#include <cstdint>

#include "dense_la.cuh"

namespace hx {

// debug counters (jobs, sweeps) of the warp Jacobi kernels, read with HX_JAC_STATS
__device__ unsigned long long g_jac_stats[2];

// One-sided Jacobi SVD of R (q x q, column-major) with lane c holding column c of R and of
// V in registers.  Pairs follow the same round-robin (circle) ordering as the CTA kernel.
// One warp: one-sided Jacobi SVD of jb (any address space for the job's arrays).
template <int QM>
__device__ __forceinline__ void warp_jacobi_run(const JacJob& jb, int lane) {
  const int q = jb.q;
  double col[QM], vc[QM];
#pragma unroll
  for (int x = 0; x < QM; ++x) {
    col[x] = (lane < q && x < q) ? (jb.trans ? jb.R[lane + x * q] : jb.R[x + lane * q]) : 0.0;
    vc[x] = (x == lane && lane < q) ? 1.0 : 0.0;
  }
  const int qe = (q + 1) & ~1;
  const double tol = 1e-15;
  int sweep = 0;
  for (; sweep < 60 && q > 1; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < qe - 1; ++r) {
      // partner of this lane in round r (circle method; position 0 is fixed)
      int partner = -1;
      if (lane < qe) {
        // lane's position on the circle
        int pos;
        if (lane == 0) {
          pos = 0;
        } else {
          pos = ((lane - 1 - r) % (qe - 1) + (qe - 1)) % (qe - 1) + 1;
        }
        int ppos;
        if (pos == 0) ppos = 1;
        else if (pos == 1) ppos = 0;
        else ppos = qe + 1 - pos;
        partner = (ppos == 0) ? 0 : ((ppos - 1 + r) % (qe - 1)) + 1;
      }
      const int src = (partner >= 0 && partner < 32) ? partner : lane;
      double pc[QM];
#pragma unroll
      for (int x = 0; x < QM; ++x) pc[x] = __shfl_sync(0xffffffffu, col[x], src);
      const bool low = lane < partner;
      bool doit = false;
      double c = 1.0, s = 0.0;
      if (lane < q && partner >= 0 && partner < q) {
        double a = 0.0, b = 0.0, g = 0.0;
#pragma unroll
        for (int x = 0; x < QM; ++x) {
          const double u = low ? col[x] : pc[x];
          const double w = low ? pc[x] : col[x];
          a += u * u;
          b += w * w;
          g += u * w;
        }
        if (fabs(g) > tol * sqrt(a * b) && g != 0.0) {
          const double zeta = (b - a) / (2.0 * g);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          c = 1.0 / sqrt(1.0 + t * t);
          s = c * t;
          doit = true;
          rotated = 1;
        }
      }
      // low column i: c*mi - s*mj ; high column j: s*mi + c*mj  (same for V)
#pragma unroll
      for (int x = 0; x < QM; ++x) {
        const double pvx = __shfl_sync(0xffffffffu, vc[x], src);
        if (doit) {
          col[x] = low ? c * col[x] - s * pc[x] : s * pc[x] + c * col[x];
          vc[x] = low ? c * vc[x] - s * pvx : s * pvx + c * vc[x];
        }
      }
    }
    if (!__any_sync(0xffffffffu, rotated)) break;
  }
  if (lane == 0) {
    atomicAdd(&g_jac_stats[0], 1ull);
    atomicAdd(&g_jac_stats[1], (unsigned long long)sweep);
  }
  // singular values = column norms; descending order (stable) via ranking by all lanes
  double nrm = 0.0;
#pragma unroll
  for (int x = 0; x < QM; ++x) nrm += col[x] * col[x];
  nrm = (lane < q) ? sqrt(nrm) : -1.0;
  int pos = 0;
  for (int d = 0; d < q; ++d) {
    const double od = __shfl_sync(0xffffffffu, nrm, d);
    if (od > nrm || (od == nrm && d < lane)) ++pos;
  }
  if (lane < q) {
    jb.sig[pos] = nrm;
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    double* col_out = jb.trans ? jb.V : jb.W;
    double* rot_out = jb.trans ? jb.W : jb.V;
#pragma unroll
    for (int x = 0; x < QM; ++x)
      if (x < q) {
        col_out[x + pos * q] = nrm > 0.0 ? col[x] * inv : 0.0;
        rot_out[x + pos * q] = vc[x];
      }
  }
}

template <int QM>
__global__ void __launch_bounds__(128) warp_jacobi_kernel(const JacJob* __restrict__ jobs,
                                                          int n_jobs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int jid = blockIdx.x * (blockDim.x >> 5) + warp;
  if (jid >= n_jobs) return;
  warp_jacobi_run<QM>(jobs[jid], lane);
}

}  // namespace hx

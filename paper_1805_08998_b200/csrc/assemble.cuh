// GPU operand assembly: assemble_hmatrix (/root/reference/pkg/src/hmat/hmatrix.py:97-118).
// Included by runtime.cu (single translation unit).
//
//   near leaves          dense kernel blocks (kernel_block, geometry.py:157-187, unit weights)
//   far leaves           partially pivoted ACA on kernel entries (aca, compressors.py:162-247):
//                        start row 0, column pivot = argmax |residual row| over unused
//                        columns, next row = argmax |residual column| over unused rows,
//                        zero-row skip (<= 1e-14 ||LU||), null-cross stop (<= 1e-15 ||LU||),
//                        two consecutive negligible crosses end the iteration, incremental
//                        ||LU||_F^2; rank > 1 results get the exact SVD recompression at
//                        eps/2 (truncate, lowrank.py:107-113) via QR + QR + Jacobi.
//   degraded far leaves  (rows exhausted without a certified zero) stored dense, flagged
// One CTA per far leaf for the cross iteration; the recompression reuses the batched QR /
// Jacobi / select kernels of the product.

namespace hx {

struct AcaJob {
  int r0, c0, m, n, kcap;
  double* L;      // m x kcap, ld m
  double* U;      // n x kcap, ld n
  uint8_t* used;  // m + n flags
};

struct DenseJob {
  int r0, c0, m, n;
  double* dst;    // m x n column-major
};

struct CopyJob {
  const double* src;
  double* dst;
  int64_t n;
};

__device__ __forceinline__ double kernel_entry(int kernel, const double* __restrict__ x,
                                               const double* __restrict__ y, int dim, double h) {
  double d2 = 0.0;
  for (int a = 0; a < dim; ++a) {
    const double t = __dsub_rn(x[a], y[a]);
    d2 = __dadd_rn(d2, __dmul_rn(t, t));
  }
  const double r = sqrt(d2);
  switch (kernel) {
    case 0: return exp(-r);
    case 1: return exp(-r / 0.5);
    case 2: return exp(-__dmul_rn(r, r) / 0.1);
    default: return 1.0 / (r + h);
  }
}

// block-wide argmax of (v, i): larger v wins, ties go to the smaller index (np.argmax)
__device__ void block_argmax(double& v, int& i, double* sv, int* si) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (ov > v || (ov == v && oi < i)) {
      v = ov;
      i = oi;
    }
  }
  __syncthreads();
  if (lane == 0) {
    sv[warp] = v;
    si[warp] = i;
  }
  __syncthreads();
  v = sv[0];
  i = si[0];
  const int nw = blockDim.x >> 5;
  for (int w = 1; w < nw; ++w)
    if (sv[w] > v || (sv[w] == v && si[w] < i)) {
      v = sv[w];
      i = si[w];
    }
}

__global__ void __launch_bounds__(LA_THREADS) aca_kernel(const AcaJob* __restrict__ jobs,
                                                         const double* __restrict__ pts, int dim,
                                                         int kernel, double h, double eps,
                                                         int* __restrict__ rank_out,
                                                         int* __restrict__ deg_out) {
  __shared__ double red[LA_THREADS / 32];
  __shared__ double sv[LA_THREADS / 32];
  __shared__ int si[LA_THREADS / 32];
  __shared__ double coef[JAC_QMAX];
  const AcaJob jb = jobs[blockIdx.x];
  const int m = jb.m, n = jb.n, tid = threadIdx.x, nt = blockDim.x;
  uint8_t* used_r = jb.used;
  uint8_t* used_c = jb.used + m;
  for (int x = tid; x < m + n; x += nt) jb.used[x] = 0;
  __syncthreads();
  const int kcap = min(jb.kcap, min(m, n));
  int k = 0, piv = 0, zero_rows = 0, hits = 0, degraded = 0;
  double norm_sq = 0.0;
  const double* X = pts + int64_t(jb.r0) * dim;
  const double* Yp = pts + int64_t(jb.c0) * dim;
  while (k < kcap) {
    if (piv < 0 || used_r[piv]) {
      double v = -1.0;
      int idx = 0x7fffffff;
      for (int x = tid; x < m; x += nt)
        if (!used_r[x]) {
          v = 0.0;
          idx = min(idx, x);
        }
      // smallest free row: maximise v (0 for free rows), ties -> smallest index
      block_argmax(v, idx, sv, si);
      if (v < 0.0) {
        degraded = !(k == 0 && zero_rows == m);
        break;
      }
      piv = idx;
    }
    __syncthreads();
    if (tid == 0) used_r[piv] = 1;
    for (int q = tid; q < k; q += nt) coef[q] = jb.L[piv + int64_t(q) * m];
    __syncthreads();
    // residual row -> U[:, k]
    double* u = jb.U + int64_t(k) * n;
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int j = tid; j < n; j += nt) {
      double v = kernel_entry(kernel, X + int64_t(piv) * dim, Yp + int64_t(j) * dim, dim, h);
      for (int q = 0; q < k; ++q) v -= jb.U[j + int64_t(q) * n] * coef[q];
      u[j] = v;
      const double a = used_c[j] ? 0.0 : fabs(v);
      if (a > bv || (a == bv && j < bi)) {
        bv = a;
        bi = j;
      }
    }
    block_argmax(bv, bi, sv, si);
    const int jc = bi;
    const double mag = bv;
    const double scale = sqrt(norm_sq);
    if (mag <= 1e-14 * scale || mag == 0.0) {
      if (k > 0) break;
      ++zero_rows;
      piv = -1;
      __syncthreads();
      continue;
    }
    __syncthreads();
    const double pivot = u[jc];
    __syncthreads();
    double nu2 = 0.0;
    for (int j = tid; j < n; j += nt) {
      const double w = u[j] / pivot;
      u[j] = w;
      nu2 += w * w;
    }
    for (int q = tid; q < k; q += nt) coef[q] = jb.U[jc + int64_t(q) * n];
    __syncthreads();
    nu2 = block_sum(nu2, red);
    // residual column -> L[:, k]
    double* l = jb.L + int64_t(k) * m;
    double nl2 = 0.0;
    for (int i = tid; i < m; i += nt) {
      double v = kernel_entry(kernel, X + int64_t(i) * dim, Yp + int64_t(jc) * dim, dim, h);
      for (int q = 0; q < k; ++q) v -= jb.L[i + int64_t(q) * m] * coef[q];
      l[i] = v;
      nl2 += v * v;
    }
    nl2 = block_sum(nl2, red);
    const double nl = sqrt(nl2), nu = sqrt(nu2);
    const double upd = nl * nu;
    if (upd <= 1e-15 * scale || upd == 0.0) break;
    if (eps > 0.0) {
      const double acc = k ? scale : upd;
      hits = (nl * nu <= eps * acc) ? hits + 1 : 0;
    }
    if (tid == 0) used_c[jc] = 1;
    // cross term sum_q (L_q . l)(U_q . u)
    double cross = 0.0;
    {
      const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
      for (int q = warp; q < k; q += nw) {
        double a = 0.0, b = 0.0;
        for (int i = lane; i < m; i += 32) a += jb.L[i + int64_t(q) * m] * l[i];
        for (int j = lane; j < n; j += 32) b += jb.U[j + int64_t(q) * n] * u[j];
        a = warp_sum(a);
        b = warp_sum(b);
        if (lane == 0) cross += a * b;
      }
    }
    cross = block_sum(cross, red);
    norm_sq += 2.0 * cross + upd * upd;
    ++k;
    if (hits >= 2) break;
    // next pivot row: argmax |l| over unused rows, none if all zero
    __syncthreads();
    double lv = 0.0;
    int li = 0x7fffffff;
    for (int i = tid; i < m; i += nt) {
      const double a = used_r[i] ? 0.0 : fabs(l[i]);
      if (a > lv || (a == lv && i < li)) {
        lv = a;
        li = i;
      }
    }
    block_argmax(lv, li, sv, si);
    piv = (lv > 0.0) ? li : -1;
    __syncthreads();
  }
  if (tid == 0) {
    rank_out[blockIdx.x] = k;
    // stopping at the workspace cap without the two-hit criterion is not a certified
    // approximation: store the block dense like a degraded one
    deg_out[blockIdx.x] = degraded || (k == kcap && kcap < min(m, n) && hits < 2);
  }
}

__global__ void dense_block_kernel(const DenseJob* __restrict__ jobs,
                                   const double* __restrict__ pts, int dim, int kernel, double h) {
  const DenseJob jb = jobs[blockIdx.x];
  const int64_t total = int64_t(jb.m) * jb.n;
  for (int64_t e = blockIdx.y * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.y) * blockDim.x) {
    const int i = int(e % jb.m), j = int(e / jb.m);
    jb.dst[e] = kernel_entry(kernel, pts + int64_t(jb.r0 + i) * dim,
                             pts + int64_t(jb.c0 + j) * dim, dim, h);
  }
}

__global__ void copy_kernel(const CopyJob* __restrict__ jobs) {
  const CopyJob jb = jobs[blockIdx.x];
  for (int64_t e = threadIdx.x; e < jb.n; e += blockDim.x) jb.dst[e] = jb.src[e];
}

}  // namespace hx

// Far leaves are processed in batches whose cross workspace fits a fixed budget; each
// batch's recompressed factors are stashed compactly, and the final pool is laid out once
// every rank is known.
extern "C" int hx_assemble(hx_ctx* c, const hx_tree* tree, const double* points, int dim,
                           int kernel, double h, double eps, int8_t* payload, int32_t* rank,
                           int64_t* u_off, int64_t* v_off, int64_t* d_off, int8_t* degraded,
                           double** pool_dev, int64_t* pool_elems) {
  using hx::panel_layout;
  return guarded([&]() -> int {
    if (!c || !tree || !points || !payload || !rank || !u_off || !v_off || !d_off ||
        !degraded || !pool_dev || !pool_elems)
      return fail(HX_EINVAL, "null argument");
    if (dim < 1 || dim > 3) return fail(HX_EINVAL, "points must be 1-, 2- or 3-dimensional");
    if (kernel < 0 || kernel > 3) return fail(HX_EINVAL, "unknown kernel id");
    if (!(eps > 0.0)) return fail(HX_EINVAL, "eps must be positive");
    CK(cudaSetDevice(c->device));
    cudaStream_t s = c->s;
    const int nn = tree->n_nodes;
    const int64_t npts = tree->c_hi[0] - tree->c_lo[0];
    DArr<double> dpts;
    dpts.upload(points, size_t(npts * dim), s);
    std::vector<int> far;
    for (int b = 0; b < nn; ++b) {
      payload[b] = 0;
      rank[b] = 0;
      u_off[b] = v_off[b] = d_off[b] = 0;
      degraded[b] = 0;
      if (tree->kind[b] == 1) far.push_back(b);
    }
    auto lo = [&](int cl) { return tree->c_lo[cl]; };
    auto sz = [&](int cl) { return tree->c_hi[cl] - tree->c_lo[cl]; };
    auto a16 = [](int64_t x) { return (x + 15) & ~int64_t(15); };
    const int kglob = JAC_QMAX;
    const size_t nf = far.size();
    std::vector<int> far_rank(nf, 0), far_deg(nf, 0), fin_rank(nf, 0);
    // compact per-leaf results: left (m x r) then right (n x r) in a stash buffer
    std::vector<DArr<double>> stash;
    std::vector<int> stash_id(nf, -1);
    std::vector<int64_t> stash_off(nf, 0);
    const int64_t WS_BUDGET = int64_t(1) << 30;  // doubles of cross workspace per batch
    struct Slots {
      double *L, *U, *RL, *RU, *core, *W, *V, *sig;
      int m, n, kc;
    };
    DArr<double> ws;
    DArr<AcaJob> daj;
    DArr<int> drank, ddeg;
    DArr<CopyJob> dcj;
    size_t f0 = 0;
    while (f0 < nf) {
      // ---- batch [f0, f1) within the workspace budget
      size_t f1 = f0;
      int64_t ws_total = 0;
      std::vector<int64_t> ws_off;
      while (f1 < nf) {
        const int b = far[f1];
        const int64_t m = sz(tree->tau[b]), n = sz(tree->sigma[b]);
        const int64_t kc = std::min<int64_t>(kglob, std::min(m, n));
        const int64_t need = a16((m + n) * kc + 5 * kc * kc + kc) + a16((m + n + 7) / 8 + 1);
        if (f1 > f0 && ws_total + need > WS_BUDGET) break;
        ws_off.push_back(ws_total);
        ws_total += need;
        ++f1;
      }
      const size_t nb = f1 - f0;
      ws.ensure(size_t(std::max<int64_t>(ws_total, 16)));
      std::vector<AcaJob> aj(nb);
      std::vector<Slots> sl(nb);
      for (size_t q = 0; q < nb; ++q) {
        const int b = far[f0 + q];
        Slots& x = sl[q];
        x.m = int(sz(tree->tau[b]));
        x.n = int(sz(tree->sigma[b]));
        x.kc = std::min(kglob, std::min(x.m, x.n));
        double* p = ws.p + ws_off[q];
        x.L = p;
        p += int64_t(x.m) * x.kc;
        x.U = p;
        p += int64_t(x.n) * x.kc;
        x.RL = p;
        p += int64_t(x.kc) * x.kc;
        x.RU = p;
        p += int64_t(x.kc) * x.kc;
        x.core = p;
        p += int64_t(x.kc) * x.kc;
        x.W = p;
        p += int64_t(x.kc) * x.kc;
        x.V = p;
        p += int64_t(x.kc) * x.kc;
        x.sig = p;
        p += x.kc;
        aj[q] = AcaJob{int(lo(tree->tau[b])), int(lo(tree->sigma[b])), x.m, x.n, x.kc, x.L, x.U,
                       reinterpret_cast<uint8_t*>(ws.p + ws_off[q] +
                                                  a16((int64_t(x.m) + x.n) * x.kc +
                                                      5 * int64_t(x.kc) * x.kc + x.kc))};
      }
      daj.upload(aj, s);
      drank.ensure(nb);
      ddeg.ensure(nb);
      aca_kernel<<<int(nb), LA_THREADS, 0, s>>>(daj.p, dpts.p, dim, kernel, h, eps, drank.p,
                                                ddeg.p);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(far_rank.data() + f0, drank.p, nb * sizeof(int), cudaMemcpyDeviceToHost,
                         s));
      CK(cudaMemcpyAsync(far_deg.data() + f0, ddeg.p, nb * sizeof(int), cudaMemcpyDeviceToHost,
                         s));
      CK(cudaStreamSynchronize(s));
      // ---- eps/2 recompression of rank > 1 crosses (truncate / lowrank_svd)
      std::vector<int> tr;
      for (size_t q = 0; q < nb; ++q) {
        fin_rank[f0 + q] = far_rank[f0 + q];
        if (!far_deg[f0 + q] && far_rank[f0 + q] > 1) tr.push_back(int(q));
      }
      if (!tr.empty()) {
        std::vector<QrJob> qj;
        for (int q : tr) {
          qj.push_back(QrJob{sl[q].L, sl[q].RL, sl[q].m, far_rank[f0 + q]});
          qj.push_back(QrJob{sl[q].U, sl[q].RU, sl[q].n, far_rank[f0 + q]});
        }
        run_qr(c, qj);
        double* saved_work = c->own[BUF_WORK].p;
        c->own[BUF_WORK].p = ws.p;
        std::vector<Term> tt;
        std::vector<Tile> tl;
        std::vector<Group> tg;
        for (int q : tr) {
          const int k = far_rank[f0 + q];
          single_term_tiles(tt, tl, tg,
                            mk(BUF_WORK, sl[q].RL - ws.p, k, 0, BUF_WORK, sl[q].RU - ws.p, k, 0, k,
                               k, k),
                            BUF_WORK, sl[q].core - ws.p, k, k);
        }
        run_gemm_batch(c, tt, tl, tg);
        c->own[BUF_WORK].p = saved_work;
        std::vector<JacJob> jj;
        for (int q : tr)
          jj.push_back(JacJob{sl[q].core, sl[q].sig, sl[q].W, sl[q].V, far_rank[f0 + q]});
        run_jacobi(c, jj);
        std::vector<SelJob> sj;
        for (int q : tr)
          sj.push_back(SelJob{sl[q].sig, nullptr, far_rank[f0 + q], far_rank[f0 + q], 1, 0});
        const int nt = int(tr.size());
        c->sel_jobs.upload(sj, s);
        c->rank_d.ensure(size_t(nt));
        c->retry_d.ensure(size_t(nt));
        select_rank_kernel<<<(nt + 127) / 128, 128, 0, s>>>(c->sel_jobs.p, nt, 0, 0.5 * eps, 0,
                                                            1, c->rank_d.p, c->retry_d.p);
        CK(cudaGetLastError());
        std::vector<int> rk(nt);
        CK(cudaMemcpyAsync(rk.data(), c->rank_d.p, nt * sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (int a = 0; a < nt; ++a) fin_rank[f0 + tr[a]] = rk[a];
      }
      // ---- compact factors of this batch into a stash buffer
      int64_t st_total = 0;
      for (size_t q = 0; q < nb; ++q) {
        const size_t f = f0 + q;
        if (far_deg[f] || fin_rank[f] == 0) continue;
        stash_off[f] = st_total;
        st_total += a16(int64_t(sl[q].m) * fin_rank[f]) + a16(int64_t(sl[q].n) * fin_rank[f]);
      }
      if (st_total > 0) {
        stash.emplace_back();
        DArr<double>& sb = stash.back();
        sb.ensure(size_t(st_total));
        const int sid = int(stash.size() - 1);
        std::vector<SmallJob> jl;
        std::vector<CopyJob> cj;
        int qmax = 1, rows_max = 1;
        for (size_t q = 0; q < nb; ++q) {
          const size_t f = f0 + q;
          if (far_deg[f] || fin_rank[f] == 0) continue;
          stash_id[f] = sid;
          const Slots& x = sl[q];
          const int r = fin_rank[f];
          double* left = sb.p + stash_off[f];
          double* right = left + a16(int64_t(x.m) * r);
          if (far_rank[f] <= 1) {
            cj.push_back(CopyJob{x.L, left, int64_t(x.m) * r});
            cj.push_back(CopyJob{x.U, right, int64_t(x.n) * r});
          } else {
            const int k = far_rank[f];
            jl.push_back(SmallJob{x.L, x.W, x.sig, left, x.m, k, k, x.m, r});
            jl.push_back(SmallJob{x.U, x.V, nullptr, right, x.n, k, k, x.n, r});
            qmax = std::max(qmax, k);
            rows_max = std::max(rows_max, std::max(x.m, x.n));
          }
        }
        if (!cj.empty()) {
          dcj.upload(cj, s);
          copy_kernel<<<int(cj.size()), 256, 0, s>>>(dcj.p);
          CK(cudaGetLastError());
        }
        if (!jl.empty()) {
          c->small_jobs.upload(jl, s);
          dim3 grid(unsigned(jl.size()), unsigned(std::min(8, (rows_max + 127) / 128)));
          small_product_kernel<<<grid, 128, 0, s>>>(c->small_jobs.p);
          CK(cudaGetLastError());
        }
        CK(cudaStreamSynchronize(s));  // job arrays and the workspace are reused next batch
      }
      f0 = f1;
    }
    ws.release();
    // ---- final pool layout: panel order (see panel_layout)
    std::vector<int> far_index(nn, -1);
    for (size_t f = 0; f < nf; ++f) far_index[far[f]] = int(f);
    for (int b = 0; b < nn; ++b) {
      if (tree->kind[b] == 0) continue;
      const int f = far_index[b];
      if (f >= 0 && !far_deg[f]) {
        payload[b] = 1;
        rank[b] = fin_rank[f];
      } else {
        payload[b] = 2;
        if (f >= 0) degraded[b] = 1;
      }
    }
    const int64_t pos = panel_layout(tree, payload, rank, u_off, v_off, d_off);
    double* pool = nullptr;
    if (cudaMalloc(&pool, size_t(std::max<int64_t>(pos, 16)) * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      throw hx::OutOfMemory("operand pool");
    }
    c->pools.push_back(pool);
    // dense payloads (near leaves and degraded far leaves)
    std::vector<DenseJob> dj;
    int64_t max_elems = 1;
    for (int b = 0; b < nn; ++b) {
      if (payload[b] != 2) continue;
      const int m = int(sz(tree->tau[b])), n = int(sz(tree->sigma[b]));
      dj.push_back(DenseJob{int(lo(tree->tau[b])), int(lo(tree->sigma[b])), m, n, pool + d_off[b]});
      max_elems = std::max<int64_t>(max_elems, int64_t(m) * n);
    }
    DArr<DenseJob> ddj;
    if (!dj.empty()) {
      ddj.upload(dj, s);
      dim3 grid(unsigned(dj.size()), unsigned(std::min<int64_t>(64, (max_elems + 255) / 256)));
      dense_block_kernel<<<grid, 256, 0, s>>>(ddj.p, dpts.p, dim, kernel, h);
      CK(cudaGetLastError());
    }
    // low-rank payloads from the stash
    std::vector<CopyJob> cj;
    for (size_t f = 0; f < nf; ++f) {
      const int b = far[f];
      if (payload[b] != 1 || rank[b] == 0) continue;
      const int64_t m = sz(tree->tau[b]), n = sz(tree->sigma[b]);
      const double* left = stash[size_t(stash_id[f])].p + stash_off[f];
      const double* right = left + a16(m * rank[b]);
      cj.push_back(CopyJob{left, pool + u_off[b], m * rank[b]});
      cj.push_back(CopyJob{right, pool + v_off[b], n * rank[b]});
    }
    if (!cj.empty()) {
      dcj.upload(cj, s);
      copy_kernel<<<int(cj.size()), 256, 0, s>>>(dcj.p);
      CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(s));
    for (auto& sb : stash) sb.release();
    dpts.release();
    daj.release();
    drank.release();
    ddeg.release();
    ddj.release();
    dcj.release();
    *pool_dev = pool;
    *pool_elems = pos;
    return HX_OK;
  });
}

extern "C" int hx_pool_download(hx_ctx* c, const double* pool, double* host, int64_t n) {
  return guarded([&]() -> int {
    if (!c || !pool || !host || n < 0) return fail(HX_EINVAL, "bad arguments");
    CK(cudaSetDevice(c->device));
    // cudaMemcpyDefault: the destination may be host memory or another device buffer
    CK(cudaMemcpyAsync(host, pool, size_t(n) * sizeof(double), cudaMemcpyDefault, c->s));
    CK(cudaStreamSynchronize(c->s));
    return HX_OK;
  });
}

extern "C" int hx_pool_free(hx_ctx* c, double* pool) {
  return guarded([&]() -> int {
    if (!c || !pool) return fail(HX_EINVAL, "bad arguments");
    auto it = std::find(c->pools.begin(), c->pools.end(), pool);
    if (it == c->pools.end()) return fail(HX_EINVAL, "not a pool of this context");
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->s));
    cudaFree(pool);
    c->pools.erase(it);
    return HX_OK;
  });
}

// Traditional-mode executor (host side): the wave loop over the conversion trees built by
// plan.cpp (see traditional.cuh for the design).  Included by runtime.cu after the batched
// QR / Jacobi / GEMM helpers it drives.
#pragma once
#include <array>

namespace {

using hx::TNode;
using hx::TNormJob;
using hx::TSeg;
using hx::TVal;

// One truncation T(sum of inputs) on an m x n block; inputs on sub-blocks at (ro, co).
struct TJob {
  int node;
  int m, n;
  std::vector<std::pair<int, std::array<int, 4>>> in;  // (value id, {ro, co, mc, nc})
  bool final_ = false;
  // workspace (doubles, offsets in the wave workspace)
  int K = 0, a = 0, b = 0, q = 0;
  bool qrl = false, qrr = false;
  int64_t xl = 0, xr = 0, rl = 0, rr = 0, core = 0, w = 0, v = 0, sg = 0;
};

TVal term_value(const BufPtrs& bp, const Term& tm, int64_t row0, int64_t col0) {
  if (tm.b_kc > 1 || tm.a_kc > 1) throw hx::Unsupported("gathered term in traditional mode");
  TVal x;
  const int64_t ri = row0 - tm.r_lo, ci = col0 - tm.c_lo;
  const double* A = bp.p[tm.a_buf] + tm.a_off;
  const double* B = bp.p[tm.b_buf] + tm.b_off;
  x.L = tm.a_kc ? A + ri * tm.a_ld : A + ri;
  x.lrow = int8_t(tm.a_kc);
  x.ldl = tm.a_ld;
  x.R = tm.b_kc ? B + ci * tm.b_ld : B + ci;
  x.rrow = int8_t(tm.b_kc);
  x.ldr = tm.b_ld;
  x.k = tm.k;
  return x;
}

// Far leaves of a traditional-mode plan; fills f.direct / f.Y / f.Bt / f.rank of every far
// block and returns the reference's matvec count (compressor converters only).
int64_t run_traditional(hx_ctx* c, hx_plan* P, const hx_product_cfg* cfg,
                        std::vector<FarBlock>& fb, int& waves) {
  const BufPtrs bp = c->ptrs();
  cudaStream_t s = c->s;
  std::vector<TNode> nodes(P->tnodes.begin(), P->tnodes.end());
  std::vector<std::vector<int32_t>> kids(nodes.size());
  for (size_t i = 0; i < nodes.size(); ++i)
    kids[i].assign(P->tkids.begin() + nodes[i].kid_begin, P->tkids.begin() + nodes[i].kid_end);
  // the inherited terms of each leaf (its root path) become items of the leaf root, ahead
  // of the converted pairs (multiply.py:217-218)
  for (const FarBlock& f : fb) {
    const OutLeaf& L = P->leaves[size_t(f.leaf)];
    if (L.troot < 0) throw std::runtime_error("far leaf without a traditional-mode root");
    std::vector<int32_t> path;
    for (int32_t g = L.g_begin; g < L.g_end; ++g) {
      const Group gr = P->mat_groups[size_t(g)];
      for (int32_t ti = gr.t_begin; ti < gr.t_end; ++ti) {
        if (P->mat_terms[size_t(ti)].k <= 0) continue;
        TNode x{};
        x.kind = hx::TN_LR;
        x.term = ti;
        x.m = L.m;
        x.n = L.n;
        x.row0 = L.row0;
        x.col0 = L.col0;
        path.push_back(int32_t(nodes.size()));
        nodes.push_back(x);
        kids.emplace_back();
      }
    }
    auto& rk = kids[size_t(L.troot)];
    rk.insert(rk.begin(), path.begin(), path.end());
  }
  const int nn = int(nodes.size());
  std::vector<int> parent(nn, -1), pending(nn, 0);
  for (int i = 0; i < nn; ++i)
    for (int k : kids[i]) {
      parent[k] = i;
      if (nodes[k].kind >= hx::TN_FOLD) pending[i]++;
    }
  std::vector<TVal> val(nn);
  std::vector<TNormJob> nj;
  c->trad_nv.ensure(size_t(std::max(nn, 1)));
  for (int i = 0; i < nn; ++i) {
    if (nodes[i].kind >= hx::TN_FOLD) continue;
    val[i] = term_value(bp, P->mat_terms[size_t(nodes[i].term)], nodes[i].row0, nodes[i].col0);
    const int p = parent[i];
    if (p >= 0 && nodes[p].sort)
      nj.push_back(TNormJob{val[i].L, val[i].R, val[i].ldl, val[i].ldr, nodes[i].m, nodes[i].n,
                            val[i].k, val[i].lrow, val[i].rrow, c->trad_nv.p + i});
  }
  if (!nj.empty()) {  // sort keys of the leaf roots' items
    c->trad_norm_jobs.upload(nj, s);
    hx::trad_norm_kernel<<<int(nj.size()), 256, 0, s>>>(c->trad_norm_jobs.p);
    CK(cudaGetLastError());
    c->launches++;
    std::vector<double> nv(static_cast<size_t>(nn));
    c->d2h(nv.data(), c->trad_nv.p, size_t(nn) * sizeof(double), s);
    for (int i = 0; i < nn; ++i)
      if (nodes[i].kind < hx::TN_FOLD) val[i].norm = nv[size_t(i)];
  }

  // fold states
  std::vector<std::vector<int32_t>> order(nn);
  std::vector<size_t> pos(nn, 0);
  std::vector<TVal> acc(nn);
  std::vector<int> active, next;
  for (int i = 0; i < nn; ++i)
    if (nodes[i].kind >= hx::TN_FOLD && pending[i] == 0) active.push_back(i);
  c->trad_release(false);
  auto a16 = [](int64_t x) { return (x + 15) & ~int64_t(15); };
  waves = 0;
  int parity = 0;
  std::vector<TJob> jobs;
  while (!active.empty()) {
    jobs.clear();
    next.clear();
    auto finish = [&](int f, const TVal& v) {
      val[f] = v;
      const int p = parent[f];
      if (p >= 0 && --pending[p] == 0) next.push_back(p);
    };
    for (int f : active) {
      const TNode& nd = nodes[f];
      TJob j;
      j.node = f;
      j.m = nd.m;
      j.n = nd.n;
      auto add_in = [&](int v) {
        const TNode& x = nodes[v];
        j.in.push_back({v, {int(x.row0 - nd.row0), int(x.col0 - nd.col0), x.m, x.n}});
      };
      if (pos[f] == 0 && order[f].empty()) {
        for (int k : kids[f])
          if (val[k].k > 0) order[f].push_back(k);
        if (nd.sort)
          std::stable_sort(order[f].begin(), order[f].end(),
                           [&](int x, int y) { return val[x].norm > val[y].norm; });
        if (order[f].empty()) {  // nothing of rank > 0: the zero block
          finish(f, TVal{});
          continue;
        }
        if (nd.kind == hx::TN_STACK) {
          for (int k : order[f]) add_in(k);
          pos[f] = order[f].size();
        } else {
          add_in(order[f][0]);
          if (order[f].size() > 1) add_in(order[f][1]);
          pos[f] = std::min<size_t>(2, order[f].size());
        }
      } else {
        j.in.push_back({-1 - f, {0, 0, nd.m, nd.n}});  // the running sum
        add_in(order[f][pos[f]]);
        pos[f]++;
      }
      j.final_ = pos[f] >= order[f].size();
      jobs.push_back(std::move(j));
    }
    if (jobs.empty()) {
      active.swap(next);
      continue;
    }
    ++waves;
    auto value_of = [&](int v) -> const TVal& { return v >= 0 ? val[size_t(v)] : acc[size_t(-1 - v)]; };
    // ---- workspace layout
    int64_t ws = 0;
    for (TJob& j : jobs) {
      j.K = 0;
      for (auto& in : j.in) j.K += value_of(in.first).k;
      j.qrl = j.K < j.m;
      j.qrr = j.K < j.n;
      j.a = j.qrl ? j.K : j.m;
      j.b = j.qrr ? j.K : j.n;
      j.q = std::max(j.a, j.b);
      if (j.q > hx::JAC_QMAX)
        throw hx::Unsupported("traditional mode: truncation core wider than " +
                              std::to_string(hx::JAC_QMAX));
      const int64_t K = j.K, q = j.q;
      j.xl = ws;
      ws = a16(ws + j.m * K);
      j.xr = ws;
      ws = a16(ws + j.n * K);
      j.rl = ws;
      if (j.qrl) ws = a16(ws + K * K);
      j.rr = ws;
      if (j.qrr) ws = a16(ws + K * K);
      j.core = ws;
      ws = a16(ws + q * q);
      j.w = ws;
      ws = a16(ws + q * q);
      j.v = ws;
      ws = a16(ws + q * q);
      j.sg = ws;
      ws = a16(ws + q);
    }
    c->trad_ws.ensure(size_t(std::max<int64_t>(ws, 1)));
    double* W0 = c->trad_ws.p;
    // ---- gather
    std::vector<TSeg> segs;
    int64_t seg_max = 1;
    for (const TJob& j : jobs) {
      int koff = 0;
      for (auto& in : j.in) {
        const TVal& x = value_of(in.first);
        if (x.k <= 0) continue;
        const auto& g = in.second;
        segs.push_back(TSeg{x.L, W0 + j.xl + int64_t(koff) * j.m, x.ldl, j.m, g[0], g[2], j.m,
                            x.k, x.lrow});
        segs.push_back(TSeg{x.R, W0 + j.xr + int64_t(koff) * j.n, x.ldr, j.n, g[1], g[3], j.n,
                            x.k, x.rrow});
        seg_max = std::max<int64_t>(seg_max, int64_t(std::max(j.m, j.n)) * x.k);
        koff += x.k;
      }
    }
    c->trad_segs.upload(segs, s);
    {
      dim3 grid(unsigned(segs.size()), unsigned(std::min<int64_t>(16, (seg_max + 1023) / 1024)));
      hx::trad_gather_kernel<<<grid, 256, 0, s>>>(c->trad_segs.p);
      CK(cudaGetLastError());
      c->launches++;
    }
    // ---- QR of the panels taller than K
    std::vector<QrJob> qj;
    for (const TJob& j : jobs) {
      if (j.qrl) qj.push_back(QrJob{W0 + j.xl, W0 + j.rl, j.m, j.K});
      if (j.qrr) qj.push_back(QrJob{W0 + j.xr, W0 + j.rr, j.n, j.K});
    }
    run_qr(c, qj);
    // ---- cores C = R_L R_R^T (zero outside a x b)
    {
      double* saved = c->own[BUF_WORK].p;
      c->own[BUF_WORK].p = W0;
      std::vector<Term> tt;
      std::vector<Tile> tl;
      std::vector<Group> tg;
      for (const TJob& j : jobs) {
        const int64_t lo = j.qrl ? j.rl : j.xl, ro = j.qrr ? j.rr : j.xr;
        const int lld = j.qrl ? j.K : j.m, rld = j.qrr ? j.K : j.n;
        single_term_tiles(tt, tl, tg, mk(BUF_WORK, lo, lld, 0, BUF_WORK, ro, rld, 0, j.K, j.a, j.b),
                          BUF_WORK, j.core, j.q, j.q);
      }
      run_gemm_batch(c, tt, tl, tg);
      c->own[BUF_WORK].p = saved;
    }
    // ---- SVD of the cores and the rank
    std::vector<JacJob> jj;
    std::vector<SelJob> sj;
    std::vector<const double*> sigp;
    for (const TJob& j : jobs) {
      jj.push_back(JacJob{W0 + j.core, W0 + j.sg, W0 + j.w, W0 + j.v, j.q, 0});
      const int l = std::min(j.a, j.b);
      sj.push_back(SelJob{W0 + j.sg, nullptr, l, l, 1, 0});
      sigp.push_back(W0 + j.sg);
    }
    run_jacobi(c, jj);
    const int na = int(jobs.size());
    c->sel_jobs.upload(sj, s);
    c->rank_d.ensure(size_t(na));
    c->retry_d.ensure(size_t(na));
    select_rank_kernel<<<(na + 127) / 128, 128, 0, s>>>(c->sel_jobs.p, na, cfg->policy, cfg->eps,
                                                        cfg->k_max, 0, c->rank_d.p, c->retry_d.p);
    CK(cudaGetLastError());
    c->trad_sigp.upload(sigp, s);
    c->trad_nv.ensure(size_t(std::max(nn, na)));
    hx::trad_sig_norm_kernel<<<(na + 127) / 128, 128, 0, s>>>(c->trad_sigp.p, c->rank_d.p,
                                                              c->trad_nv.p, na);
    CK(cudaGetLastError());
    c->launches += 2;
    std::vector<int> rk(static_cast<size_t>(na));
    std::vector<double> nrm(static_cast<size_t>(na));
    c->d2h(rk.data(), c->rank_d.p, size_t(na) * sizeof(int), s);
    c->d2h(nrm.data(), c->trad_nv.p, size_t(na) * sizeof(double), s);
    // ---- outputs: running sums in this wave's ping-pong arena, finished values kept
    int64_t tmp_sz = 0, keep_sz = 0;
    std::vector<int64_t> off(static_cast<size_t>(na));
    for (int i = 0; i < na; ++i) {
      const TJob& j = jobs[size_t(i)];
      int64_t& sz = j.final_ ? keep_sz : tmp_sz;
      off[size_t(i)] = sz;
      sz = a16(sz + int64_t(j.m + j.n) * rk[size_t(i)]);
    }
    c->trad_tmp[parity].ensure(size_t(std::max<int64_t>(tmp_sz, 1)));
    double* keep = nullptr;
    if (keep_sz > 0) {
      c->trad_keep.emplace_back();
      c->trad_keep.back().ensure(size_t(keep_sz));
      keep = c->trad_keep.back().p;
    }
    std::vector<SmallJob> jl;
    int rows_max = 1;
    for (int i = 0; i < na; ++i) {
      const TJob& j = jobs[size_t(i)];
      const int r = rk[size_t(i)];
      TVal o;
      o.k = r;
      o.norm = nrm[size_t(i)];
      if (r > 0) {
        double* base = (j.final_ ? keep : c->trad_tmp[parity].p) + off[size_t(i)];
        double* ol = base;
        double* orr = base + int64_t(j.m) * r;
        if (j.qrl)
          jl.push_back(SmallJob{W0 + j.xl, W0 + j.w, W0 + j.sg, ol, j.m, j.a, j.q, j.m, r});
        else
          jl.push_back(SmallJob{nullptr, W0 + j.w, W0 + j.sg, ol, j.m, j.a, j.q, 0, r});
        if (j.qrr)
          jl.push_back(SmallJob{W0 + j.xr, W0 + j.v, nullptr, orr, j.n, j.b, j.q, j.n, r});
        else
          jl.push_back(SmallJob{nullptr, W0 + j.v, nullptr, orr, j.n, j.b, j.q, 0, r});
        o.L = ol;
        o.R = orr;
        o.ldl = j.m;
        o.ldr = j.n;
        rows_max = std::max(rows_max, std::max(j.m, j.n));
      }
      if (j.final_)
        finish(j.node, o);
      else
        acc[size_t(j.node)] = o;
    }
    if (!jl.empty()) {
      c->small_jobs.upload(jl, s);
      dim3 grid(unsigned(jl.size()), unsigned(std::min(8, (rows_max + 127) / 128)));
      small_product_kernel<<<grid, 128, 0, s>>>(c->small_jobs.p);
      CK(cudaGetLastError());
      c->launches++;
    }
    for (const TJob& j : jobs)
      if (!j.final_) next.push_back(j.node);
    active.swap(next);
    parity ^= 1;
  }
  for (FarBlock& f : fb) {
    const TVal& v = val[size_t(P->leaves[size_t(f.leaf)].troot)];
    f.direct = 1;
    f.rank = v.k;
    f.Y = const_cast<double*>(v.L);
    f.Bt = const_cast<double*>(v.R);
    f.done = 1;
  }
  return P->trad_matvecs;
}

}  // namespace

// Flat term-list builder: the restrict/_thin_product bookkeeping of the reference product,
// restated as one DFS over the block-cluster tree that emits device work lists.
//
// Reference semantics followed (file:line in /root/reference/pkg/src/hmat):
//   sumexpr_root            sumexpr.py:78-83   S(I x I) = {(A_root, B_root)}
//   restrict                sumexpr.py:136-154 low-rank terms are inherited by slicing,
//                                              pending pairs split over the middle cluster
//   _split_pair             sumexpr.py:120-133 inner pair -> sub-pairs (tau' x rho', rho' x sigma')
//   _thin_product           sumexpr.py:93-117  far x far: core = V_A^T U_B, smaller rank pushed
//                                              far x X : (U_A, X^T V_A);  X x far : (X U_B, V_B)
//   rank-0 terms dropped    sumexpr.py:150
//   _node_matmat            hmatrix.py:177-202 X U_B / X^T V_A as sums over the leaves of X
//   evaluate_dense / the compressors see  S = sum U_j V_j^T + sum P Q;  pending inner x inner
//   pairs at far leaves are expanded into the same kinds of terms on sub-blocks (exact,
//   SURVEY Appendix D), pending near x near pairs become dense x dense products.
//
// Every created term has one computed factor, and it is always "an H-block times a thin
// matrix":  left_t = X U  (X = the A-side block, U = U_B)  or  right_t = X^T V  (X = the
// B-side block, V = V_A) -- far x far pushes the smaller rank, which is the same formula
// with X a single low-rank leaf.  Terms sharing the same X (on average ~35 on config 2)
// are batched: their thin factors are gathered side by side into G and X is applied once
// to G, so X's leaves are read once per group instead of once per term.
//
// Output: batches for the device
//   gather: thin factors copied into each group's G
//   core  : V_l^T G (A side) / U_l^T G (B side) for the low-rank leaves l of X
//   fac   : row bands of X G / X^T G  (dense leaves D_l G, low-rank leaves U_l core_l)
//   mat   : every output leaf materialized tile by tile from the terms of its root path
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hx.h"
#include "hx_internal.h"

using hx::Group;
using hx::Term;
using hx::Tile;

namespace {

constexpr int INNER = 0, FAR = 1, NEAR = 2;

inline int64_t align16(int64_t x) { return (x + 15) & ~int64_t(15); }

// One created low-rank term (before batching).
struct TRec {
  int32_t pc, qc;    // A-side and B-side blocks of the sub-pair
  int32_t k;         // rank of the term
  int32_t mat;       // index of its materialization term (patched with the factor offset)
  int8_t side;       // 0: left_t = X U_B (X = pc), 1: right_t = X^T V_A (X = qc)
};

struct Builder {
  const hx_tree& t;
  const hx_operand& A;
  const hx_operand& B;
  const uint8_t* mask;
  int T;
  hx_plan& P;
  std::vector<uint8_t> owned_sub;
  std::vector<TRec> recs;

  // materialization groups of the current root path (real blocks)
  std::vector<int32_t> path_groups;

  struct VGroup {
    int32_t g;  // index into group table (term range)
    int64_t r0, r1, c0, c1;
  };

  Builder(const hx_tree& t_, const hx_operand& a, const hx_operand& b, const uint8_t* m,
          int tile, hx_plan& plan)
      : t(t_), A(a), B(b), mask(m), T(tile), P(plan) {}

  int64_t lo(int c) const { return t.c_lo[c]; }
  int64_t sz(int c) const { return t.c_hi[c] - t.c_lo[c]; }
  int kind(int b) const { return t.kind[b]; }
  bool isF(const hx_operand& op, int b) const { return t.kind[b] == FAR && op.payload[b] == 1; }
  bool isD(const hx_operand& op, int b) const {
    return t.kind[b] == NEAR || (t.kind[b] == FAR && op.payload[b] == 2);
  }
  int child_of(int b, int i, int j) const { return t.child[4 * b + 2 * i + j]; }

  static Term make_term(uint8_t abuf, int64_t aoff, int32_t ald, uint8_t akc, uint8_t bbuf,
                        int64_t boff, int32_t bld, uint8_t bkc, int32_t k, int64_t rlo,
                        int64_t clo, int64_t rows, int64_t cols) {
    Term x;
    x.a_off = aoff;
    x.b_off = boff;
    x.a_ld = ald;
    x.b_ld = bld;
    x.k = k;
    x.r_lo = int32_t(rlo);
    x.c_lo = int32_t(clo);
    x.rows = int32_t(rows);
    x.cols = int32_t(cols);
    x.a_buf = abuf;
    x.b_buf = bbuf;
    x.a_kc = akc;
    x.b_kc = bkc;
    return x;
  }

  // Tiles over an R x C output (column-major, ld = R) at out_off in out_buf; the tile grid
  // starts at coordinate (row_base, 0).  `band_pieces[i]` are the terms of row band i.
  void emit_band_tiles(std::vector<Term>& terms, std::vector<Tile>& tiles,
                       std::vector<Group>& groups, uint8_t out_buf, int64_t out_off, int64_t R,
                       int64_t C, int64_t row_base,
                       const std::vector<std::vector<Term>>& band_pieces) {
    for (int64_t i = 0, band = 0; i < R; i += T, ++band) {
      const int64_t r1 = std::min<int64_t>(R, i + T);
      const int32_t gb = int32_t(terms.size());
      for (const Term& p : band_pieces[band]) terms.push_back(p);
      const int32_t gidx = int32_t(groups.size());
      groups.push_back(Group{gb, int32_t(terms.size())});
      for (int64_t j = 0; j < C; j += T) {
        Tile tl;
        std::memset(&tl, 0, sizeof(tl));
        tl.out_off = out_off + i + j * R;
        tl.out_ld = int32_t(R);
        tl.row0 = int32_t(row_base + i);
        tl.col0 = int32_t(j);
        tl.rows = int16_t(r1 - i);
        tl.cols = int16_t(std::min<int64_t>(C, j + T) - j);
        tl.g_begin = gidx;
        tl.g_end = gidx + 1;
        tl.aux = -1;
        tl.out_buf = out_buf;
        tl.mode = hx::MODE_STORE;
        tiles.push_back(tl);
      }
    }
  }

  // Leaves of the subtree of node x (DFS order), with the multiply/byte counts of one
  // thin product through it (hmatrix.py:177-202).
  void subtree_leaves(const hx_operand& op, int x, std::vector<int>& out, double& mv,
                      double& bytes) {
    if (kind(x) == INNER) {
      for (int c = 0; c < 4; ++c) {
        const int ch = t.child[4 * x + c];
        if (ch >= 0) subtree_leaves(op, ch, out, mv, bytes);
      }
      return;
    }
    const double m = double(sz(t.tau[x])), n = double(sz(t.sigma[x]));
    if (isF(op, x)) {
      const double k = op.rank[x];
      mv += 2.0 * k * (m + n);
      bytes += 8.0 * k * (m + n);
    } else {
      mv += 2.0 * m * n;
      bytes += 8.0 * m * n;
    }
    out.push_back(x);
  }

  // --------------------------------------------------------------- term creation
  // One sub-pair (pc, qc) on the (real or virtual) block tc x sc with a factored side:
  // _thin_product (sumexpr.py:93-117).  Records the term; its computed factor is produced
  // by the group pass.  Returns the rank of the new term (0 = dropped).
  int create_lr(int tc, int sc, int pc, int qc, int log_block) {
    const int64_t m = sz(tc), n = sz(sc);
    const bool aF = isF(A, pc), bF = isF(B, qc);
    int k, kind_log;
    int8_t side;
    if (aF && bF) {
      const int kA = A.rank[pc], kB = B.rank[qc];
      if (kA == 0 || kB == 0) return 0;
      kind_log = 0;
      if (kA <= kB) {
        side = 1;  // (U_A, V_B core^T): right = B_qc^T V_A
        k = kA;
      } else {
        side = 0;  // (U_A core, V_B): left = A_pc U_B
        k = kB;
      }
    } else if (aF) {
      k = A.rank[pc];
      if (k == 0) return 0;
      side = 1;
      kind_log = 1;
    } else {
      k = B.rank[qc];
      if (k == 0) return 0;
      side = 0;
      kind_log = 2;
    }
    TRec r;
    r.pc = pc;
    r.qc = qc;
    r.k = k;
    r.side = side;
    r.mat = int32_t(P.mat_terms.size());
    recs.push_back(r);
    // the fixed factor is a pool factor; the computed one is patched by build_groups()
    if (side == 0)
      P.mat_terms.push_back(make_term(hx::BUF_TERM, -1, int32_t(m), 0, hx::BUF_B, B.v_off[qc],
                                      int32_t(n), 0, k, lo(tc), lo(sc), m, n));
    else
      P.mat_terms.push_back(make_term(hx::BUF_A, A.u_off[pc], int32_t(m), 0, hx::BUF_TERM, -1,
                                      int32_t(n), 0, k, lo(tc), lo(sc), m, n));
    if (log_block >= 0) log(log_block, kind_log, pc, qc, k);
    return k;
  }

  void create_dxd(int tc, int sc, int pc, int qc) {
    const int rho = t.sigma[pc];
    const int64_t m = sz(tc), n = sz(sc), kr = sz(rho);
    if (!isD(A, pc) || !isD(B, qc))
      throw hx::Unsupported("pending pair that is neither inner x inner nor dense x dense");
    if (t.tau[pc] != tc || t.sigma[qc] != sc)
      throw hx::Unsupported("dense sub-views (ragged cluster trees)");
    P.mat_terms.push_back(make_term(hx::BUF_A, A.d_off[pc], int32_t(m), 0, hx::BUF_B,
                                    B.d_off[qc], int32_t(kr), 1, int32_t(kr), lo(tc), lo(sc),
                                    m, n));
    P.info.n_dxd++;
  }

  void log(int block, int k, int a, int b, int r) {
    P.log_block.push_back(block);
    P.log_kind.push_back(int8_t(k));
    P.log_a.push_back(a);
    P.log_b.push_back(b);
    P.log_rank.push_back(r);
    P.info.created[k]++;
  }

  // --------------------------------------------------------------- grouped term factors
  // workspace bound (doubles) for one batch of gathered factors, and for its cores
  static constexpr int64_t budget = int64_t(1) << 28;

  void build_groups() {
    const int nn = t.n_nodes;
    const size_t nr = recs.size();
    // counting sort of the terms by (side, X)
    std::vector<int32_t> cnt(2 * size_t(nn) + 1, 0);
    auto key = [&](const TRec& r) { return r.side * nn + (r.side == 0 ? r.pc : r.qc); };
    for (const TRec& r : recs) cnt[key(r) + 1]++;
    for (size_t i = 1; i < cnt.size(); ++i) cnt[i] += cnt[i - 1];
    std::vector<int32_t> order(nr);
    {
      std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
      for (size_t i = 0; i < nr; ++i) order[pos[key(recs[i])]++] = int32_t(i);
    }
    std::vector<int> leaves;
    std::vector<std::vector<Term>> bands;
    int64_t gat_cur = 0, core_cur = 0;
    auto close_batch = [&]() {
      hx_plan::Batch& bt = P.batches.back();
      bt.gather_end = int64_t(P.gather.size());
      bt.core_end = int64_t(P.core_tiles.size());
      bt.fac_end = int64_t(P.fac_tiles.size());
    };
    auto open_batch = [&]() {
      P.batches.push_back(hx_plan::Batch{int64_t(P.gather.size()), 0,
                                         int64_t(P.core_tiles.size()), 0,
                                         int64_t(P.fac_tiles.size()), 0});
      gat_cur = 0;
      core_cur = 0;
    };
    open_batch();
    for (int g = 0; g < 2 * nn; ++g) {
      const int32_t b0 = cnt[g], b1 = cnt[g + 1];
      if (b0 == b1) continue;
      const int side = g >= nn ? 1 : 0;
      const int X = g - side * nn;
      const hx_operand& opX = side == 0 ? A : B;
      // rows of the computed factor and of the middle cluster rho'
      const int rows_cl = side == 0 ? t.tau[X] : t.sigma[X];
      const int rho = side == 0 ? t.sigma[X] : t.tau[X];
      const int64_t R = sz(rows_cl), kr = sz(rho);
      int64_t ktot = 0;
      for (int32_t i = b0; i < b1; ++i) ktot += recs[order[i]].k;
      leaves.clear();
      double mv = 0, bytes = 0;
      subtree_leaves(opX, X, leaves, mv, bytes);
      int64_t core_need = 0;
      for (int l : leaves)
        if (isF(opX, l)) core_need += align16(int64_t(opX.rank[l]) * ktot);
      const int64_t gat_need = align16(kr * ktot);
      if ((gat_cur + gat_need > budget || core_cur + core_need > budget) &&
          (gat_cur > 0 || core_cur > 0)) {
        close_batch();
        open_batch();
      }
      const int64_t out = P.term_elems;
      P.term_elems = align16(P.term_elems + R * ktot);
      const int64_t gat = gat_cur;
      gat_cur += gat_need;
      P.gather_elems = std::max(P.gather_elems, gat_cur);
      // gather the thin factors side by side, patch the materialization terms
      int64_t col = 0;
      for (int32_t i = b0; i < b1; ++i) {
        const TRec& r = recs[order[i]];
        hx::CopyRec cp;
        cp.src_buf = side == 0 ? hx::BUF_B : hx::BUF_A;
        cp.src_off = side == 0 ? B.u_off[r.qc] : A.v_off[r.pc];
        cp.dst_off = gat + col * kr;
        cp.n = kr * r.k;
        P.gather.push_back(cp);
        Term& mt = P.mat_terms[r.mat];
        if (side == 0) {
          mt.a_off = out + col * R;
          mt.a_ld = int32_t(R);
        } else {
          mt.b_off = out + col * R;
          mt.b_ld = int32_t(R);
        }
        col += r.k;
      }
      // X applied to G: leaves of X
      P.info.flops_form += double(ktot) * mv;
      P.info.bytes_form += double(b1 - b0) * bytes + 8.0 * double(ktot) * double(kr + R);
      P.info.n_xgroups++;
      const int64_t nb = (R + T - 1) / T;
      bands.assign(size_t(nb), {});
      for (int l : leaves) {
        // A side: leaf l = (tau_l, rho_l) rows tau_l;  B side: l = (rho_l, sigma_l) rows sigma_l
        const int rl = side == 0 ? t.sigma[l] : t.tau[l];   // middle-cluster part
        const int ol = side == 0 ? t.tau[l] : t.sigma[l];   // output rows
        const int64_t roff = lo(rl) - lo(rho);
        Term piece;
        if (isF(opX, l)) {
          const int kl = opX.rank[l];
          if (kl == 0) continue;
          // core_l = V_l^T G[rho_l] (A side) or U_l^T G[rho_l] (B side): kl x ktot
          const int64_t core = core_cur;
          core_cur = align16(core_cur + int64_t(kl) * ktot);
          P.core_elems = std::max(P.core_elems, core_cur);
          const int64_t mid_f = side == 0 ? opX.v_off[l] : opX.u_off[l];
          std::vector<std::vector<Term>> one(size_t((kl + T - 1) / T));
          const Term cp = make_term(side == 0 ? hx::BUF_A : hx::BUF_B, mid_f, int32_t(sz(rl)), 1,
                                    hx::BUF_GATHER, gat + roff, int32_t(kr), 1, int32_t(sz(rl)),
                                    0, 0, kl, ktot);
          for (auto& v : one) v.push_back(cp);
          emit_band_tiles(P.core_terms, P.core_tiles, P.core_groups, hx::BUF_CORE, core, kl, ktot,
                          0, one);
          const int64_t out_f = side == 0 ? opX.u_off[l] : opX.v_off[l];
          piece = make_term(side == 0 ? hx::BUF_A : hx::BUF_B, out_f, int32_t(sz(ol)), 0,
                            hx::BUF_CORE, core, kl, 1, kl, lo(ol), 0, sz(ol), ktot);
        } else {
          // dense: D_l G[rho_l] (A side) or D_l^T G[rho_l] (B side)
          piece = make_term(side == 0 ? hx::BUF_A : hx::BUF_B, opX.d_off[l], int32_t(sz(t.tau[l])),
                            uint8_t(side == 0 ? 0 : 1), hx::BUF_GATHER, gat + roff, int32_t(kr), 1,
                            int32_t(sz(rl)), lo(ol), 0, sz(ol), ktot);
        }
        const int64_t a = (lo(ol) - lo(rows_cl)) / T;
        const int64_t e = (lo(ol) + sz(ol) - lo(rows_cl) - 1) / T;
        for (int64_t bnd = std::max<int64_t>(a, 0); bnd <= std::min<int64_t>(e, nb - 1); ++bnd)
          bands[size_t(bnd)].push_back(piece);
      }
      emit_band_tiles(P.fac_terms, P.fac_tiles, P.fac_groups, hx::BUF_TERM, out, R, ktot,
                      lo(rows_cl), bands);
    }
    close_batch();
  }

  // --------------------------------------------------------------- the descent
  // Pending pairs of (virtual) block tc x sc split onto child (ti, si):
  // sumexpr.py:146-153.  Created terms are appended to P.mat_terms (current group).
  void split_pairs(int tc, int sc, int ti, int si, const std::vector<std::pair<int, int>>& pend,
                   std::vector<std::pair<int, int>>& sub, int log_block, int64_t& K) {
    const int tcc = t.c_child[2 * tc + ti], scc = t.c_child[2 * sc + si];
    for (const auto& pq : pend) {
      const int p = pq.first, q = pq.second;
      if (kind(p) != INNER || kind(q) != INNER)
        throw hx::Unsupported("pending pair with a dense side above the leaf level");
      for (int ri = 0; ri < 2; ++ri) {
        const int pc = child_of(p, ti, ri), qc = child_of(q, ri, si);
        if (pc < 0 || qc < 0) throw std::runtime_error("block tree is not level-conserving");
        if (isF(A, pc) || isF(B, qc)) {
          K += create_lr(tcc, scc, pc, qc, log_block);
        } else {
          sub.emplace_back(pc, qc);
        }
      }
    }
  }

  // Expansion of the pending inner x inner pairs of a far leaf over virtual sub-blocks
  // (exact).
  void expand(int tc, int sc, const std::vector<std::pair<int, int>>& pend,
              std::vector<VGroup>& vg, int64_t& K, double& fdd, double& edd) {
    if (pend.empty()) return;
    if (t.c_child[2 * tc] < 0 || t.c_child[2 * sc] < 0)
      throw std::runtime_error("expand reached leaf clusters");
    for (int ti = 0; ti < 2; ++ti)
      for (int si = 0; si < 2; ++si) {
        const int tcc = t.c_child[2 * tc + ti], scc = t.c_child[2 * sc + si];
        const int32_t gb = int32_t(P.mat_terms.size());
        std::vector<std::pair<int, int>> sub;
        int64_t Kv = 0;
        split_pairs(tc, sc, ti, si, pend, sub, -1, Kv);
        K += Kv;
        P.info.n_terms_expand += int64_t(P.mat_terms.size()) - gb;
        const bool leaf_level = t.c_child[2 * tcc] < 0 || t.c_child[2 * scc] < 0;
        if (leaf_level) {
          for (const auto& pq : sub) {
            create_dxd(tcc, scc, pq.first, pq.second);
            const double mm = double(sz(tcc)), nn = double(sz(scc)),
                         kk = double(sz(t.sigma[pq.first]));
            fdd += 2.0 * mm * kk * nn;
            edd += mm * kk + kk * nn;
          }
        }
        const int32_t ge = int32_t(P.mat_terms.size());
        if (ge > gb) {
          P.mat_groups_all.push_back(Group{gb, ge});
          vg.push_back(VGroup{int32_t(P.mat_groups_all.size() - 1), lo(tcc), lo(tcc) + sz(tcc),
                              lo(scc), lo(scc) + sz(scc)});
        }
        if (!leaf_level) expand(tcc, scc, sub, vg, K, fdd, edd);
      }
  }

  void emit_leaf_tiles(int b, bool far, const std::vector<VGroup>& vg, int64_t K, double fdd,
                       double edd) {
    const int tc = t.tau[b], sc = t.sigma[b];
    const int64_t m = sz(tc), n = sz(sc);
    hx::OutLeaf L;
    L.id = b;
    L.kind = far ? 1 : 2;
    L.m = int32_t(m);
    L.n = int32_t(n);
    L.row0 = lo(tc);
    L.col0 = lo(sc);
    int64_t& ws = far ? ws_far : ws_near;
    L.ws_off = ws;
    L.K = K;
    L.fdd = fdd;
    L.edd = edd;
    ws = align16(ws + m * n);
    L.tile_begin = int32_t(P.mat_tiles.size());
    L.sumsq_begin = P.n_sumsq;
    int32_t prev_gb = -1, prev_ge = -1;
    std::vector<int32_t> cur, prev;
    for (int64_t j = 0; j < n; j += T) {
      for (int64_t i = 0; i < m; i += T) {
        const int64_t r0 = lo(tc) + i, r1 = lo(tc) + std::min<int64_t>(m, i + T);
        const int64_t c0 = lo(sc) + j, c1 = lo(sc) + std::min<int64_t>(n, j + T);
        cur.assign(path_groups.begin(), path_groups.end());
        for (const VGroup& v : vg)
          if (v.r0 < r1 && v.r1 > r0 && v.c0 < c1 && v.c1 > c0) cur.push_back(v.g);
        int32_t gb, ge;
        if (cur == prev) {
          gb = prev_gb;
          ge = prev_ge;
        } else {
          gb = int32_t(P.mat_groups.size());
          for (int32_t g : cur) P.mat_groups.push_back(P.mat_groups_all[g]);
          ge = int32_t(P.mat_groups.size());
          prev = cur;
          prev_gb = gb;
          prev_ge = ge;
        }
        Tile tl;
        std::memset(&tl, 0, sizeof(tl));
        tl.out_off = L.ws_off + i + j * m;
        tl.out_ld = int32_t(m);
        tl.row0 = int32_t(r0);
        tl.col0 = int32_t(c0);
        tl.rows = int16_t(r1 - r0);
        tl.cols = int16_t(c1 - c0);
        tl.g_begin = gb;
        tl.g_end = ge;
        tl.out_buf = hx::BUF_TILE;
        tl.mode = hx::MODE_STORE_SUMSQ;
        tl.aux = P.n_sumsq++;
        P.mat_tiles.push_back(tl);
      }
    }
    L.tile_end = int32_t(P.mat_tiles.size());
    L.sumsq_end = P.n_sumsq;
    P.info.max_out_dim = std::max<int64_t>(P.info.max_out_dim, std::max(m, n));
    P.leaves.push_back(L);
  }

  int64_t path_K = 0;
  int64_t ws_far = 0, ws_near = 0;

  void visit(int b, const std::vector<std::pair<int, int>>& pend) {
    const int tc = t.tau[b], sc = t.sigma[b];
    for (int ci = 0; ci < 4; ++ci) {
      const int c = t.child[4 * b + ci];
      if (c < 0 || !owned_sub[c]) continue;
      const int32_t gb = int32_t(P.mat_terms.size());
      std::vector<std::pair<int, int>> sub;
      int64_t Kc = 0;
      split_pairs(tc, sc, ci >> 1, ci & 1, pend, sub, c, Kc);
      P.info.n_terms_real += int64_t(P.mat_terms.size()) - gb;
      // DxD pairs of a leaf at the leaf level join the leaf's own group
      const bool leaf_level = kind(c) != INNER &&
                              (t.c_child[2 * t.tau[c]] < 0 || t.c_child[2 * t.sigma[c]] < 0);
      double fdd = 0, edd = 0;
      std::vector<std::pair<int, int>> rest;
      if (leaf_level) {
        for (const auto& pq : sub) {
          create_dxd(t.tau[c], t.sigma[c], pq.first, pq.second);
          const double mm = double(sz(t.tau[c])), nn = double(sz(t.sigma[c])),
                       kk = double(sz(t.sigma[pq.first]));
          fdd += 2.0 * mm * kk * nn;
          edd += mm * kk + kk * nn;
        }
      } else {
        rest.swap(sub);
      }
      const int32_t ge = int32_t(P.mat_terms.size());
      const bool has = ge > gb;
      if (has) {
        P.mat_groups_all.push_back(Group{gb, ge});
        path_groups.push_back(int32_t(P.mat_groups_all.size() - 1));
      }
      const int64_t save_K = path_K;
      path_K += Kc;
      if (kind(c) == INNER) {
        visit(c, rest);
      } else {
        std::vector<VGroup> vg;
        int64_t K = path_K;
        if (kind(c) == FAR) expand(t.tau[c], t.sigma[c], rest, vg, K, fdd, edd);
        else if (!rest.empty()) throw hx::Unsupported("near leaf above the leaf level");
        const double mm = double(sz(t.tau[c])), nn = double(sz(t.sigma[c]));
        if (kind(c) == NEAR) {
          P.info.flops_near += fdd + 2.0 * mm * nn * double(K);
          P.info.bytes_near += 8.0 * (double(K) * (mm + nn) + edd + mm * nn);
          P.info.n_near++;
        } else {
          P.info.n_far++;
        }
        emit_leaf_tiles(c, kind(c) == FAR, vg, K, fdd, edd);
      }
      path_K = save_K;
      if (has) path_groups.pop_back();
    }
  }

  // near blocks go after the far ones so the result download is two contiguous copies
  void place_near() {
    P.near_ws_begin = ws_far;
    P.tile_elems = ws_far + ws_near;
    for (hx::OutLeaf& L : P.leaves) {
      if (L.kind != 2) continue;
      L.ws_off += ws_far;
      for (int32_t i = L.tile_begin; i < L.tile_end; ++i) P.mat_tiles[i].out_off += ws_far;
    }
  }

  void run() {
    const int nn = t.n_nodes;
    owned_sub.assign(nn, 0);
    // bottom-up ownership: children have larger pre-order ids than their parent
    for (int b = nn - 1; b >= 0; --b) {
      if (t.kind[b] != INNER) {
        owned_sub[b] = mask ? (mask[b] != 0) : 1;
      } else {
        uint8_t o = 0;
        for (int c = 0; c < 4; ++c) {
          const int ch = t.child[4 * b + c];
          if (ch >= 0 && owned_sub[ch]) o = 1;
        }
        owned_sub[b] = o;
      }
    }
    if (t.kind[0] != INNER) {
      // the root itself is a leaf: S(root) = {(A_root, B_root)} evaluated directly
      if (owned_sub[0]) {
        const int tc = t.tau[0], sc = t.sigma[0];
        if (t.kind[0] == FAR) throw hx::Unsupported("admissible root block");
        const int32_t gb = int32_t(P.mat_terms.size());
        create_dxd(tc, sc, 0, 0);
        P.mat_groups_all.push_back(Group{gb, int32_t(P.mat_terms.size())});
        path_groups.push_back(int32_t(P.mat_groups_all.size() - 1));
        const double m = double(sz(tc));
        const double fdd = 2.0 * m * m * m, edd = 2.0 * m * m;
        P.info.flops_near += fdd;
        P.info.bytes_near += 8.0 * (edd + m * m);
        P.info.n_near++;
        std::vector<VGroup> vg;
        emit_leaf_tiles(0, false, vg, 0, fdd, edd);
      }
    } else {
      std::vector<std::pair<int, int>> root{{0, 0}};
      visit(0, root);
    }
    build_groups();
    place_near();
  }
};

}  // namespace

extern "C" int hx_plan_create(const hx_tree* tree, const hx_operand* a, const hx_operand* b,
                              const uint8_t* leaf_mask, int tile, hx_plan** out) {
  return hx::guarded([&]() -> int {
    if (!tree || !a || !b || !out) return hx::fail(HX_EINVAL, "null argument");
    if (tile != 32 && tile != 64) return hx::fail(HX_EINVAL, "tile must be 32 or 64");
    if (tree->n_nodes <= 0 || tree->n_clusters <= 0) return hx::fail(HX_EINVAL, "empty tree");
    auto* plan = new hx_plan();
    std::memset(&plan->info, 0, sizeof(plan->info));
    plan->tile = tile;
    try {
      Builder bld(*tree, *a, *b, leaf_mask, tile, *plan);
      bld.run();
    } catch (...) {
      delete plan;
      throw;
    }
    hx_plan_info& I = plan->info;
    I.n_out = int64_t(plan->leaves.size());
    I.mat_terms = int64_t(plan->mat_terms.size());
    I.mat_tiles = int64_t(plan->mat_tiles.size());
    I.mat_groups = int64_t(plan->mat_groups.size());
    I.core_terms = int64_t(plan->core_terms.size());
    I.core_tiles = int64_t(plan->core_tiles.size());
    I.fac_terms = int64_t(plan->fac_terms.size());
    I.fac_tiles = int64_t(plan->fac_tiles.size());
    I.core_elems = plan->core_elems;
    I.term_elems = plan->term_elems;
    I.tile_elems = plan->tile_elems;
    I.gather_elems = plan->gather_elems;
    I.gather_jobs = int64_t(plan->gather.size());
    *out = plan;
    return HX_OK;
  });
}

extern "C" int hx_plan_info_get(const hx_plan* plan, hx_plan_info* info) {
  if (!plan || !info) return hx::fail(HX_EINVAL, "null argument");
  *info = plan->info;
  return HX_OK;
}

extern "C" int hx_plan_leaves(const hx_plan* plan, int32_t* ids, int8_t* kind, int32_t* m,
                              int32_t* n, int64_t* stacked_rank, double* f_dd, double* e_dd) {
  if (!plan) return hx::fail(HX_EINVAL, "null plan");
  for (size_t i = 0; i < plan->leaves.size(); ++i) {
    const hx::OutLeaf& L = plan->leaves[i];
    if (ids) ids[i] = L.id;
    if (kind) kind[i] = L.kind;
    if (m) m[i] = L.m;
    if (n) n[i] = L.n;
    if (stacked_rank) stacked_rank[i] = L.K;
    if (f_dd) f_dd[i] = L.fdd;
    if (e_dd) e_dd[i] = L.edd;
  }
  return HX_OK;
}

extern "C" int hx_plan_term_log(const hx_plan* plan, int32_t* block, int8_t* kind,
                                int32_t* a_node, int32_t* b_node, int32_t* rank) {
  if (!plan) return hx::fail(HX_EINVAL, "null plan");
  if (block) std::copy(plan->log_block.begin(), plan->log_block.end(), block);
  if (kind) std::copy(plan->log_kind.begin(), plan->log_kind.end(), kind);
  if (a_node) std::copy(plan->log_a.begin(), plan->log_a.end(), a_node);
  if (b_node) std::copy(plan->log_b.begin(), plan->log_b.end(), b_node);
  if (rank) std::copy(plan->log_rank.begin(), plan->log_rank.end(), rank);
  return HX_OK;
}

extern "C" void hx_plan_free(hx_plan* plan) { delete plan; }

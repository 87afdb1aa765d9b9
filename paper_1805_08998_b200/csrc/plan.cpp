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
// The descent runs sequentially down to a cut level, then the subtrees below the cut in
// parallel (OpenMP), each into its own output that is merged in DFS order; the grouped
// factor work is then counted and filled in parallel.
//
// Output: batches for the device
//   gather: thin factors copied into each group's G
//   core  : V_l^T G (A side) / U_l^T G (B side) for the low-rank leaves l of X (stacked)
//   fac   : row bands of X G / X^T G  (dense leaves D_l G, low-rank leaves U_l core_l)
//   mat   : every output leaf materialized tile by tile from the terms of its root path
#include <nvtx3/nvToolsExt.h>
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
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
  int8_t dg;         // 1: the thin matrix is a dense block (H-block x dense pair), 0: a factor
};


using PairList = std::vector<std::pair<int, int>>;
using GRef = std::pair<int32_t, int32_t>;  // (output index, group id local to that output)

// Output of one descent task (the top part or one subtree below the cut).
struct Out {
  hx::pvec<TRec> recs;
  std::vector<Term> terms;        // materialization terms
  std::vector<Group> groups;      // one per creation block (real or virtual), local indices
  std::vector<GRef> tile_groups;  // per tile: the groups of its root path and sub-blocks
  std::vector<Tile> tiles;        // g_begin/g_end index tile_groups; ws offsets local
  std::vector<hx::OutLeaf> leaves;
  std::vector<hx::TSubBlock> tsub;  // offsets local to the task's far workspace
  std::vector<int32_t> log_block, log_a, log_b, log_rank;
  std::vector<int8_t> log_kind;
  int64_t n_terms_real = 0, n_terms_expand = 0, n_dxd = 0, created[3] = {0, 0, 0};
  int64_t n_mixed = 0;  // H-block x dense terms (ragged trees)
  int64_t n_far = 0, n_near = 0, max_out_dim = 0;
  double flops_near = 0, bytes_near = 0;
  int64_t ws_far = 0, ws_near = 0;
  int32_t n_sumsq = 0;
  // traditional mode: conversion trees (term / node indices local to this output)
  std::vector<hx::TNode> tnodes;
  std::vector<int32_t> tkids;
  int64_t trad_cols = 0;
};

struct Walk {
  Out& o;
  int32_t self;
  std::vector<GRef> path;  // groups of the current root path
  int64_t path_K = 0;
  // pending-pair lists of the recursion, two per depth, reused across the whole descent (a
  // fresh std::vector per visited block made the allocator a third of the descent time)
  std::vector<PairList> pool = std::vector<PairList>(512);
  PairList& scratch(int depth, int which) {
    if (size_t(2 * depth + which) >= pool.size())
      throw std::runtime_error("block tree deeper than 256 levels");
    PairList& v = pool[size_t(2 * depth + which)];
    v.clear();
    return v;
  }
};

struct Task {
  int c;
  PairList pend;
  std::vector<GRef> path;
  int64_t path_K;
  int64_t log_pos;  // top-part log length when the subtree was deferred
};

struct VGroup {
  GRef g;
  int64_t r0, r1, c0, c1;
  int32_t blk;  // T_sub block of the leaf holding this group (index into TBlk list), -1: sketched size
};

// Outermost small (materialized rather than sketched) virtual block below a far leaf.
struct TBlk {
  int64_t r0, r1, c0, c1;
  bool used;
};

struct Builder {
  const hx_tree& t;
  const hx_operand& A;
  const hx_operand& B;
  const uint8_t* mask;
  int T;
  hx_plan& P;
  std::vector<uint8_t> owned_sub;
  hx::pvec<TRec> recs;
  bool logging = false;  // HX_PLAN_LOG: keep the restrict log (parity tests)
  int trad = 0;          // HX_PLAN_TRAD: 0 new mode, 1 hierarchical pairs, 2 stacked pairs
  int64_t implicit_min = 0;  // far leaves with min(m, n) >= this take the implicit route
  // sketch width assumed by the implicit route's per-term choice (HX_SKETCH_COLS; 0 sketches
  // every sub-block term, the fully implicit route)
  double sketch_cols = std::getenv("HX_SKETCH_COLS") ? std::atof(std::getenv("HX_SKETCH_COLS"))
                                                     : 56.0;
  // stacked-core runs start on multiples of this many rows (HX_CORE_ALIGN; 1: packed)
  int64_t core_align = std::getenv("HX_CORE_ALIGN") ? std::max(1, std::atoi(std::getenv("HX_CORE_ALIGN")))
                                                    : 8;

  Builder(const hx_tree& t_, const hx_operand& a, const hx_operand& b, const uint8_t* m,
          int tile, hx_plan& plan)
      : t(t_), A(a), B(b), mask(m), T(tile), P(plan) {}

  // implicit route: a sub-block term on an h x w extent costs ~4 (h + w) L flops per unit of
  // rank to sketch (range and co-range passes, L ~ 56 columns) against 2 h w to materialize
  bool sketched_ext(double h, double wd) const { return h * wd >= 4.0 * sketch_cols * (h + wd); }

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

  // Leaves of the subtree of node x (DFS order), with the multiply/byte counts of one
  // thin product through it (hmatrix.py:177-202).
  void subtree_leaves(const hx_operand& op, int x, std::vector<int>& out, double& mv,
                      double& bytes) const {
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
  int create_lr(Walk& w, int tc, int sc, int pc, int qc, int log_block) const {
    Out& o = w.o;
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
    r.dg = 0;
    r.mat = int32_t(o.terms.size());
    o.recs.push_back(r);
    // the fixed factor is a pool factor; the computed one is patched by build_groups()
    if (side == 0)
      o.terms.push_back(make_term(hx::BUF_TERM, -1, int32_t(m), 0, hx::BUF_B, B.v_off[qc],
                                  int32_t(n), 0, k, lo(tc), lo(sc), m, n));
    else
      o.terms.push_back(make_term(hx::BUF_A, A.u_off[pc], int32_t(m), 0, hx::BUF_TERM, -1,
                                  int32_t(n), 0, k, lo(tc), lo(sc), m, n));
    if (log_block >= 0) {
      if (logging) {
        o.log_block.push_back(log_block);
        o.log_kind.push_back(int8_t(kind_log));
        o.log_a.push_back(pc);
        o.log_b.push_back(qc);
        o.log_rank.push_back(k);
      }
      o.created[kind_log]++;
    }
    return k;
  }

  // Dense x dense pair evaluated on block tc x sc: the rows tc of D_pc times the columns sc
  // of D_qc.  On ragged trees (leaves at different depths) a dense pair stays pending below
  // its own blocks and arrives here as sub-views (HBlock.subview, hmatrix.py:257-258;
  // _split_pair's dense branch, sumexpr.py:130-133): the views are column-major slices.
  void create_dxd(Walk& w, int tc, int sc, int pc, int qc) const {
    const int rho = t.sigma[pc];
    const int64_t m = sz(tc), n = sz(sc), kr = sz(rho);
    if (!isD(A, pc) || !isD(B, qc))
      throw hx::Unsupported("pending pair that is neither inner x inner nor dense x dense");
    const int tp = t.tau[pc], sq = t.sigma[qc];
    if (lo(tc) < lo(tp) || lo(tc) + m > lo(tp) + sz(tp) || lo(sc) < lo(sq) ||
        lo(sc) + n > lo(sq) + sz(sq) || t.tau[qc] != rho)
      throw std::runtime_error("dense pair does not cover the block");
    const int64_t a_off = A.d_off[pc] + (lo(tc) - lo(tp));
    const int64_t b_off = B.d_off[qc] + (lo(sc) - lo(sq)) * kr;
    w.o.terms.push_back(make_term(hx::BUF_A, a_off, int32_t(sz(tp)), 0, hx::BUF_B, b_off,
                                  int32_t(kr), 1, int32_t(kr), lo(tc), lo(sc), m, n));
    w.o.n_dxd++;
  }

  bool dense_pair(int p, int q) const { return isD(A, p) && isD(B, q); }
  bool mixed_pair(int p, int q) const {
    return (kind(p) == INNER && isD(B, q)) || (isD(A, p) && kind(q) == INNER);
  }

  // H-block x dense pair (or dense x H-block) at a leaf-level block of a ragged tree: the
  // inner branch of _split_pair meets a leaf cluster on one side (sumexpr.py:123-129) and
  // the pair is applied through HBlock.matmat (hmatrix.py:177-211) by the compressor or
  // evaluate_dense.  Exact as a term whose computed factor is X D (or X^T D^T, D^T from a
  // transposed copy) and whose other factor is the identity.
  void create_mixed(Walk& w, int tc, int sc, int pc, int qc) const {
    Out& o = w.o;
    const int64_t m = sz(tc), n = sz(sc);
    if (t.tau[pc] != tc || t.sigma[qc] != sc || t.sigma[pc] != t.tau[qc])
      throw hx::Unsupported("H-block x dense pair on a sub-view");
    TRec r;
    r.pc = pc;
    r.qc = qc;
    r.dg = 1;
    r.mat = int32_t(o.terms.size());
    if (kind(pc) == INNER) {  // X = A_pc, thin matrix D_qc (rho x sc); right factor I
      r.k = int32_t(n);
      r.side = 0;
      o.terms.push_back(make_term(hx::BUF_TERM, -1, int32_t(m), 0, hx::BUF_EYE, 0, hx::EYE_LD, 0,
                                  int32_t(n), lo(tc), lo(sc), m, n));
    } else {  // X = B_qc, thin matrix D_pc^T (rho x tc); left factor I
      r.k = int32_t(m);
      r.side = 1;
      o.terms.push_back(make_term(hx::BUF_EYE, 0, hx::EYE_LD, 0, hx::BUF_TERM, -1, int32_t(n), 0,
                                  int32_t(m), lo(tc), lo(sc), m, n));
    }
    if (r.k > hx::EYE_LD) throw hx::Unsupported("H-block x dense pair wider than 1024");
    o.recs.push_back(r);
    o.n_mixed++;
  }

  // --------------------------------------------------------------- the descent
  // Pending pairs of (virtual) block tc x sc split onto child (ti, si):
  // sumexpr.py:146-153.  Created terms are appended to the current group.
  void split_pairs(Walk& w, int tc, int sc, int ti, int si, const PairList& pend, PairList& sub,
                   int log_block, int64_t& K) const {
    const int tcc = t.c_child[2 * tc + ti], scc = t.c_child[2 * sc + si];
    for (const auto& pq : pend) {
      const int p = pq.first, q = pq.second;
      if (dense_pair(p, q)) {
        // the middle cluster is a leaf and never splits: the pair goes down as is, its
        // views narrowing with the output block (sumexpr.py:130-133)
        sub.emplace_back(p, q);
        continue;
      }
      if (kind(p) != INNER || kind(q) != INNER)
        throw hx::Unsupported("pending pair that is neither inner x inner nor dense x dense");
      for (int ri = 0; ri < 2; ++ri) {
        const int pc = child_of(p, ti, ri), qc = child_of(q, ri, si);
        if (pc < 0 || qc < 0) throw std::runtime_error("block tree is not level-conserving");
        if (isF(A, pc) || isF(B, qc)) {
          K += create_lr(w, tcc, scc, pc, qc, log_block);
        } else {
          sub.emplace_back(pc, qc);
        }
      }
    }
  }

  // Expansion of the pending inner x inner pairs of a far leaf over virtual sub-blocks
  // (exact).
  void expand(Walk& w, int tc, int sc, const PairList& pend, std::vector<VGroup>& vg,
              int64_t& K, double& fdd, double& edd, int depth, std::vector<TBlk>& tb,
              int32_t blk_root) const {
    if (pend.empty()) return;
    if (t.c_child[2 * tc] < 0 || t.c_child[2 * sc] < 0)
      throw hx::Unsupported("H-block x dense pending pair at a leaf (ragged cluster trees)");
    Out& o = w.o;
    for (int ti = 0; ti < 2; ++ti)
      for (int si = 0; si < 2; ++si) {
        const int tcc = t.c_child[2 * tc + ti], scc = t.c_child[2 * sc + si];
        const int32_t gb = int32_t(o.terms.size());
        PairList& sub = w.scratch(depth, 0);
        int64_t Kv = 0;
        split_pairs(w, tc, sc, ti, si, pend, sub, -1, Kv);
        K += Kv;
        o.n_terms_expand += int64_t(o.terms.size()) - gb;
        const bool leaf_level = t.c_child[2 * tcc] < 0 || t.c_child[2 * scc] < 0;
        if (leaf_level) {
          for (const auto& pq : sub) {
            if (mixed_pair(pq.first, pq.second)) {
              create_mixed(w, tcc, scc, pq.first, pq.second);
              continue;
            }
            create_dxd(w, tcc, scc, pq.first, pq.second);
            const double mm = double(sz(tcc)), nn = double(sz(scc)),
                         kk = double(sz(t.sigma[pq.first]));
            fdd += 2.0 * mm * kk * nn;
            edd += mm * kk + kk * nn;
          }
        }
        const int32_t ge = int32_t(o.terms.size());
        // the outermost sub-block too small to sketch collects every group below it
        int32_t child_root = blk_root;
        if (child_root < 0 && !sketched_ext(double(sz(tcc)), double(sz(scc)))) {
          child_root = int32_t(tb.size());
          tb.push_back(TBlk{lo(tcc), lo(tcc) + sz(tcc), lo(scc), lo(scc) + sz(scc), false});
        }
        if (ge > gb) {
          o.groups.push_back(Group{gb, ge});
          vg.push_back(VGroup{GRef{w.self, int32_t(o.groups.size() - 1)}, lo(tcc),
                              lo(tcc) + sz(tcc), lo(scc), lo(scc) + sz(scc), child_root});
          if (child_root >= 0) tb[size_t(child_root)].used = true;
        }
        if (!leaf_level) expand(w, tcc, scc, sub, vg, K, fdd, edd, depth + 1, tb, child_root);
      }
  }

  void emit_leaf_tiles(Walk& w, int b, bool far, const std::vector<VGroup>& vg, int64_t K,
                       double fdd, double edd, const std::vector<TBlk>& tb) const {
    Out& o = w.o;
    const int tc = t.tau[b], sc = t.sigma[b];
    const int64_t m = sz(tc), n = sz(sc);
    hx::OutLeaf L;
    L.id = b;
    L.kind = far ? 1 : 2;
    L.m = int32_t(m);
    L.n = int32_t(n);
    L.row0 = lo(tc);
    L.col0 = lo(sc);
    int64_t& ws = far ? o.ws_far : o.ws_near;
    L.ws_off = ws;
    L.K = K;
    L.fdd = fdd;
    L.edd = edd;
    L.implicit = 0;
    L.g_begin = L.g_end = -1;
    L.troot = -1;
    L.tile_begin = int32_t(o.tiles.size());
    L.sumsq_begin = o.n_sumsq;
    // implicit route: the terms inherited from the root path (full-leaf extent, most of the
    // stacked rank of a large leaf) and the sub-block terms on large sub-blocks are only
    // sketched -- a term on an h x w extent costs ~4 (h + w) L flops per unit of rank to
    // sketch (range and co-range passes, L ~ 56 columns) against 2 h w to materialize; the
    // tiles materialize the remaining small sub-block terms into T_sub (none: no T_sub)
    const bool impl = far && implicit_min > 0 && std::min(m, n) >= implicit_min;
    L.tsub_begin = L.tsub_end = int32_t(o.tsub.size());
    if (impl) {
      L.implicit = 1;
      L.g_begin = int32_t(o.tile_groups.size());
      o.tile_groups.insert(o.tile_groups.end(), w.path.begin(), w.path.end());
      for (const VGroup& v : vg)
        if (v.blk < 0) o.tile_groups.push_back(v.g);
      L.g_end = int32_t(o.tile_groups.size());
      // T_sub: one dense block per used small sub-block, tiled like a leaf of its own; the
      // rest of the leaf (config 4's 65536-leaves: ~97 % of their 10^6 tiles) is neither
      // stored nor multiplied
      thread_local std::vector<std::vector<int32_t>> by_blk;
      if (by_blk.size() < tb.size()) by_blk.resize(tb.size());
      for (size_t q = 0; q < tb.size(); ++q) by_blk[q].clear();
      for (int32_t vi = 0; vi < int32_t(vg.size()); ++vi)
        if (vg[size_t(vi)].blk >= 0) by_blk[size_t(vg[size_t(vi)].blk)].push_back(vi);
      std::vector<GRef> cur, prev;
      for (size_t q = 0; q < tb.size(); ++q) {
        const TBlk& B = tb[q];
        if (!B.used) continue;
        const int64_t h = B.r1 - B.r0, wd = B.c1 - B.c0;
        hx::TSubBlock rec{ws, B.r0, B.c0, int32_t(h), int32_t(wd)};
        o.tsub.push_back(rec);
        int32_t prev_gb = -1, prev_ge = -1;
        prev.clear();
        for (int64_t j = 0; j < wd; j += T)
          for (int64_t i = 0; i < h; i += T) {
            const int64_t r0 = B.r0 + i, r1 = B.r0 + std::min<int64_t>(h, i + T);
            const int64_t c0 = B.c0 + j, c1 = B.c0 + std::min<int64_t>(wd, j + T);
            cur.clear();
            for (int32_t vi : by_blk[q]) {
              const VGroup& v = vg[size_t(vi)];
              if (v.r0 < r1 && v.r1 > r0 && v.c0 < c1 && v.c1 > c0) cur.push_back(v.g);
            }
            int32_t gb, ge;
            if (prev_gb >= 0 && cur == prev) {
              gb = prev_gb;
              ge = prev_ge;
            } else {
              gb = int32_t(o.tile_groups.size());
              o.tile_groups.insert(o.tile_groups.end(), cur.begin(), cur.end());
              ge = int32_t(o.tile_groups.size());
              prev = cur;
              prev_gb = gb;
              prev_ge = ge;
            }
            Tile tl;
            std::memset(&tl, 0, sizeof(tl));
            tl.out_off = rec.off + i + j * h;
            tl.out_ld = int32_t(h);
            tl.row0 = int32_t(r0);
            tl.col0 = int32_t(c0);
            tl.rows = int16_t(r1 - r0);
            tl.cols = int16_t(c1 - c0);
            tl.g_begin = gb;
            tl.g_end = ge;
            tl.out_buf = hx::BUF_TILE;
            tl.mode = hx::MODE_STORE_SUMSQ;
            tl.aux = o.n_sumsq++;
            o.tiles.push_back(tl);
          }
        ws = align16(ws + h * wd);
      }
      L.tsub_end = int32_t(o.tsub.size());
      L.tile_end = int32_t(o.tiles.size());
      L.sumsq_end = o.n_sumsq;
      o.max_out_dim = std::max<int64_t>(o.max_out_dim, std::max(m, n));
      o.leaves.push_back(L);
      return;
    }
    ws = align16(ws + m * n);
    int32_t prev_gb = -1, prev_ge = -1;
    std::vector<GRef> cur, prev;
    // sub-block groups by tile (CSR over the leaf's tile grid, column-major like the tile
    // loop; creation order kept within a tile): a scan of every group per tile is quadratic
    // on the largest leaves (config 4: 10^6 tiles x 10^4 groups per 65536-leaf)
    const int64_t nti = (m + T - 1) / T, ntj = (n + T - 1) / T;
    thread_local std::vector<int32_t> vstart, vfill, vlist;
    vstart.assign(size_t(nti * ntj) + 1, 0);
    auto tile_range = [&](const VGroup& v, int64_t& i0, int64_t& i1, int64_t& j0, int64_t& j1) {
      i0 = (v.r0 - lo(tc)) / T;
      i1 = (v.r1 - 1 - lo(tc)) / T;
      j0 = (v.c0 - lo(sc)) / T;
      j1 = (v.c1 - 1 - lo(sc)) / T;
    };
    for (const VGroup& v : vg) {
      int64_t i0, i1, j0, j1;
      tile_range(v, i0, i1, j0, j1);
      for (int64_t j = j0; j <= j1; ++j)
        for (int64_t i = i0; i <= i1; ++i) vstart[size_t(i + j * nti) + 1]++;
    }
    for (size_t k = 0; k < size_t(nti * ntj); ++k) vstart[k + 1] += vstart[k];
    vfill.assign(vstart.begin(), vstart.end() - 1);
    vlist.resize(size_t(vstart.back()));
    for (int32_t vi = 0; vi < int32_t(vg.size()); ++vi) {
      const VGroup& v = vg[size_t(vi)];
      int64_t i0, i1, j0, j1;
      tile_range(v, i0, i1, j0, j1);
      for (int64_t j = j0; j <= j1; ++j)
        for (int64_t i = i0; i <= i1; ++i) vlist[size_t(vfill[size_t(i + j * nti)]++)] = vi;
    }
    for (int64_t j = 0; j < n; j += T) {
      for (int64_t i = 0; i < m; i += T) {
        const int64_t r0 = lo(tc) + i, r1 = lo(tc) + std::min<int64_t>(m, i + T);
        const int64_t c0 = lo(sc) + j, c1 = lo(sc) + std::min<int64_t>(n, j + T);
        cur.assign(w.path.begin(), w.path.end());
        const size_t tix = size_t(i / T + (j / T) * nti);
        for (int32_t q = vstart[tix]; q < vstart[tix + 1]; ++q)
          cur.push_back(vg[size_t(vlist[size_t(q)])].g);
        int32_t gb, ge;
        if (cur == prev) {
          gb = prev_gb;
          ge = prev_ge;
        } else {
          gb = int32_t(o.tile_groups.size());
          o.tile_groups.insert(o.tile_groups.end(), cur.begin(), cur.end());
          ge = int32_t(o.tile_groups.size());
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
        tl.aux = o.n_sumsq++;
        o.tiles.push_back(tl);
      }
    }
    L.tile_end = int32_t(o.tiles.size());
    L.sumsq_end = o.n_sumsq;
    o.max_out_dim = std::max<int64_t>(o.max_out_dim, std::max(m, n));
    o.leaves.push_back(L);
  }

  // --------------------------------------------------------------- traditional mode
  int32_t add_node(Out& o, int8_t kind_, int32_t term, int tc, int sc,
                   const std::vector<int32_t>& kids, int8_t sort = 0) const {
    hx::TNode x;
    x.kind = kind_;
    x.sort = sort;
    x.term = term;
    x.m = int32_t(sz(tc));
    x.n = int32_t(sz(sc));
    x.row0 = lo(tc);
    x.col0 = lo(sc);
    x.kid_begin = int32_t(o.tkids.size());
    o.tkids.insert(o.tkids.end(), kids.begin(), kids.end());
    x.kid_end = int32_t(o.tkids.size());
    o.tnodes.push_back(x);
    return int32_t(o.tnodes.size() - 1);
  }

  // Every item of the exact expansion of the pending pair (p, q) on block tc x sc (the
  // sub-pair recursion of restrict, sumexpr.py:120-154, carried to the leaves): the terms
  // a compressor converter sees through _PairProductMap (multiply.py:82-100).
  void pair_items(Walk& w, int tc, int sc, int p, int q, std::vector<int32_t>& items) const {
    Out& o = w.o;
    if (dense_pair(p, q)) {
      const int32_t ti = int32_t(o.terms.size());
      create_dxd(w, tc, sc, p, q);
      items.push_back(add_node(o, hx::TN_DD, ti, tc, sc, {}));
      return;
    }
    if (kind(p) != INNER || kind(q) != INNER)
      throw hx::Unsupported("traditional mode: H-block x dense pending pair (ragged tree)");
    for (int ti = 0; ti < 2; ++ti)
      for (int si = 0; si < 2; ++si)
        for (int ri = 0; ri < 2; ++ri) {
          const int pc = child_of(p, ti, ri), qc = child_of(q, ri, si);
          if (pc < 0 || qc < 0) throw std::runtime_error("block tree is not level-conserving");
          const int tcc = t.tau[pc], scc = t.sigma[qc];
          if (isF(A, pc) || isF(B, qc)) {
            const int32_t tix = int32_t(o.terms.size());
            if (create_lr(w, tcc, scc, pc, qc, -1) > 0)
              items.push_back(add_node(o, hx::TN_LR, tix, tcc, scc, {}));
          } else {
            pair_items(w, tcc, scc, pc, qc, items);
          }
        }
  }

  // _convert_pair (multiply.py:192-204) of the pending pair (p, q) on block tc x sc:
  // _pair_structural_lowrank (multiply.py:140-189) -- a dense pair is one truncated SVD of
  // its product; an inner pair folds each cell (tau', sigma') over its middle children
  // (thin products as they are, inner sub-pairs recursively, dense sub-pairs by SVD) and
  // then folds the cells in row-child-major order -- or, for the stacked converter, one
  // best approximation of the whole pair product.
  int32_t trad_pair(Walk& w, int tc, int sc, int p, int q) const {
    Out& o = w.o;
    if (dense_pair(p, q)) {
      const int32_t ti = int32_t(o.terms.size());
      create_dxd(w, tc, sc, p, q);
      const int32_t item = add_node(o, hx::TN_DD, ti, tc, sc, {});
      return add_node(o, hx::TN_FOLD, -1, tc, sc, {item});  // from_dense(P Q)
    }
    if (kind(p) != INNER || kind(q) != INNER)
      throw hx::Unsupported("traditional mode: H-block x dense pending pair (ragged tree)");
    if (trad == 2) {
      std::vector<int32_t> items;
      pair_items(w, tc, sc, p, q, items);
      return add_node(o, hx::TN_STACK, -1, tc, sc, items);
    }
    std::vector<int32_t> cells;
    for (int ti = 0; ti < 2; ++ti)
      for (int si = 0; si < 2; ++si) {
        std::vector<int32_t> contrib;
        int tcc = -1, scc = -1;
        for (int ri = 0; ri < 2; ++ri) {
          const int pc = child_of(p, ti, ri), qc = child_of(q, ri, si);
          if (pc < 0 || qc < 0) throw std::runtime_error("block tree is not level-conserving");
          tcc = t.tau[pc];
          scc = t.sigma[qc];
          if (isF(A, pc) || isF(B, qc)) {
            const int32_t tix = int32_t(o.terms.size());
            if (create_lr(w, tcc, scc, pc, qc, -1) > 0)
              contrib.push_back(add_node(o, hx::TN_LR, tix, tcc, scc, {}));
          } else {
            contrib.push_back(trad_pair(w, tcc, scc, pc, qc));
          }
        }
        if (!contrib.empty()) cells.push_back(add_node(o, hx::TN_FOLD, -1, tcc, scc, contrib));
      }
    return add_node(o, hx::TN_FOLD, -1, tc, sc, cells);
  }

  // leaf_traditional (multiply.py:216-224): the leaf's inherited terms (its path groups)
  // plus one converted term per pending pair, folded in decreasing-norm order.
  void trad_leaf(Walk& w, int c, const PairList& pend) const {
    Out& o = w.o;
    const int tc = t.tau[c], sc = t.sigma[c];
    std::vector<int32_t> kids;
    for (const auto& pq : pend) {
      kids.push_back(trad_pair(w, tc, sc, pq.first, pq.second));
      if (trad == 2) o.trad_cols += sz(sc);  // dense_svd_compress applies S to n columns
    }
    hx::OutLeaf L;
    std::memset(&L, 0, sizeof(L));
    L.id = c;
    L.kind = 1;
    L.m = int32_t(sz(tc));
    L.n = int32_t(sz(sc));
    L.row0 = lo(tc);
    L.col0 = lo(sc);
    L.ws_off = o.ws_far;
    L.K = w.path_K;
    L.implicit = 0;
    L.g_begin = int32_t(o.tile_groups.size());
    o.tile_groups.insert(o.tile_groups.end(), w.path.begin(), w.path.end());
    L.g_end = int32_t(o.tile_groups.size());
    L.troot = add_node(o, hx::TN_FOLD, -1, tc, sc, kids, 1);
    L.tile_begin = L.tile_end = int32_t(o.tiles.size());
    L.sumsq_begin = L.sumsq_end = o.n_sumsq;
    o.max_out_dim = std::max<int64_t>(o.max_out_dim, std::max(sz(tc), sz(sc)));
    o.n_far++;
    o.leaves.push_back(L);
  }

  // DFS below block b (whose own terms are already created).  With `tasks`, inner children
  // at block level `cut` are deferred as parallel tasks instead of descended.
  void visit(Walk& w, int b, int level, const PairList& pend, int cut,
             std::vector<Task>* tasks) const {
    Out& o = w.o;
    const int tc = t.tau[b], sc = t.sigma[b];
    for (int ci = 0; ci < 4; ++ci) {
      const int c = t.child[4 * b + ci];
      if (c < 0 || !owned_sub[c]) continue;
      const int32_t gb = int32_t(o.terms.size());
      PairList& sub = w.scratch(level, 0);
      int64_t Kc = 0;
      split_pairs(w, tc, sc, ci >> 1, ci & 1, pend, sub, c, Kc);
      o.n_terms_real += int64_t(o.terms.size()) - gb;
      // DxD pairs of a leaf join the leaf's own group (on ragged trees as sub-views);
      // inner x inner pairs of a leaf are expanded below
      double fdd = 0, edd = 0;
      PairList& rest = w.scratch(level, 1);
      const bool trad_leaf_c = trad && kind(c) == FAR;
      if (trad_leaf_c) {
        rest.swap(sub);  // every pending pair is converted on its own (multiply.py:216-219)
      } else if (kind(c) != INNER) {
        for (const auto& pq : sub) {
          if (mixed_pair(pq.first, pq.second)) {
            create_mixed(w, t.tau[c], t.sigma[c], pq.first, pq.second);
            continue;
          }
          if (!dense_pair(pq.first, pq.second)) {
            rest.push_back(pq);
            continue;
          }
          create_dxd(w, t.tau[c], t.sigma[c], pq.first, pq.second);
          const double mm = double(sz(t.tau[c])), nn = double(sz(t.sigma[c])),
                       kk = double(sz(t.sigma[pq.first]));
          fdd += 2.0 * mm * kk * nn;
          edd += mm * kk + kk * nn;
        }
      } else {
        rest.swap(sub);
      }
      const int32_t ge = int32_t(o.terms.size());
      const bool has = ge > gb;
      if (has) {
        o.groups.push_back(Group{gb, ge});
        w.path.push_back(GRef{w.self, int32_t(o.groups.size() - 1)});
      }
      const int64_t save_K = w.path_K;
      w.path_K += Kc;
      if (kind(c) == INNER) {
        if (tasks && level + 1 >= cut) {
          tasks->push_back(Task{c, rest, w.path, w.path_K, int64_t(o.log_block.size())});
        } else {
          visit(w, c, level + 1, rest, cut, tasks);
        }
      } else if (trad_leaf_c) {
        trad_leaf(w, c, rest);
      } else {
        std::vector<VGroup> vg;
        std::vector<TBlk> tb;
        int64_t K = w.path_K;
        // inner x inner pairs pending at a leaf (far, or near above the leaf level on a
        // ragged tree) are expanded exactly over virtual sub-blocks
        expand(w, t.tau[c], t.sigma[c], rest, vg, K, fdd, edd, level + 1, tb, -1);
        const double mm = double(sz(t.tau[c])), nn = double(sz(t.sigma[c]));
        if (kind(c) == NEAR) {
          o.flops_near += fdd + 2.0 * mm * nn * double(K);
          o.bytes_near += 8.0 * (double(K) * (mm + nn) + edd + mm * nn);
          o.n_near++;
        } else {
          o.n_far++;
        }
        emit_leaf_tiles(w, c, kind(c) == FAR, vg, K, fdd, edd, tb);
      }
      w.path_K = save_K;
      if (has) w.path.pop_back();
    }
  }

  int choose_cut() const {
    // first block level holding enough owned inner blocks to keep every thread busy (a
    // masked plan -- one chunk, one rank -- owns only part of each level)
    const int want = 8 * std::max(1, omp_get_max_threads());
    std::vector<int> level_nodes{0}, next;
    for (int level = 0; level < 64 && !level_nodes.empty(); ++level) {
      int inner = 0;
      next.clear();
      for (int b : level_nodes)
        if (kind(b) == INNER && owned_sub[size_t(b)]) {
          ++inner;
          for (int c = 0; c < 4; ++c)
            if (t.child[4 * b + c] >= 0) next.push_back(t.child[4 * b + c]);
        }
      if (inner >= want) return level;
      level_nodes.swap(next);
    }
    return 1 << 30;  // small tree: no parallel tasks
  }

  // --------------------------------------------------------------- merge of the outputs
  void merge(std::vector<Out>& outs) {
    tg0 = std::chrono::steady_clock::now();
    const size_t no = outs.size();
    std::vector<int64_t> b_terms(no + 1, 0), b_tg(no + 1, 0), b_tiles(no + 1, 0),
        b_sumsq(no + 1, 0), b_far(no + 1, 0), b_near(no + 1, 0), b_recs(no + 1, 0),
        b_leaves(no + 1, 0), b_nodes(no + 1, 0), b_kids(no + 1, 0), b_tsub(no + 1, 0);
    for (size_t i = 0; i < no; ++i) {
      const Out& o = outs[i];
      b_nodes[i + 1] = b_nodes[i] + int64_t(o.tnodes.size());
      b_kids[i + 1] = b_kids[i] + int64_t(o.tkids.size());
      b_terms[i + 1] = b_terms[i] + int64_t(o.terms.size());
      b_tg[i + 1] = b_tg[i] + int64_t(o.tile_groups.size());
      b_tiles[i + 1] = b_tiles[i] + int64_t(o.tiles.size());
      b_sumsq[i + 1] = b_sumsq[i] + o.n_sumsq;
      b_far[i + 1] = b_far[i] + o.ws_far;
      b_near[i + 1] = b_near[i] + o.ws_near;
      b_recs[i + 1] = b_recs[i] + int64_t(o.recs.size());
      b_leaves[i + 1] = b_leaves[i] + int64_t(o.leaves.size());
      b_tsub[i + 1] = b_tsub[i] + int64_t(o.tsub.size());
    }
    P.mat_terms.resize(size_t(b_terms[no]));
    P.mat_groups.resize(size_t(b_tg[no]));
    P.mat_tiles.resize(size_t(b_tiles[no]));
    P.leaves.resize(size_t(b_leaves[no]));
    P.tsub.resize(size_t(b_tsub[no]));
    recs.resize(size_t(b_recs[no]));
    ws_far_total = b_far[no];
    ws_near_total = b_near[no];
    P.n_sumsq = int32_t(b_sumsq[no]);
    lap("merge alloc");
    // balanced blocks of <= 64k elements over every output array: a few tasks (the top
    // part, large subtrees) hold most of the records, so a loop over tasks alone leaves
    // most threads idle behind them
    struct Blk {
      int32_t task, what;  // what: 0 terms, 1 recs, 2 tile groups, 3 leaves (+ tiles)
      int64_t a, e;
    };
    std::vector<Blk> blks;
    constexpr int64_t BS = int64_t(1) << 16;
    for (size_t i = 0; i < no; ++i) {
      const Out& o = outs[i];
      const int64_t len[4] = {int64_t(o.terms.size()), int64_t(o.recs.size()),
                              int64_t(o.tile_groups.size()), int64_t(o.leaves.size())};
      for (int w = 0; w < 4; ++w) {
        const int64_t bs = w == 3 ? BS / 16 : BS;
        for (int64_t a = 0; a < len[w]; a += bs)
          blks.push_back(Blk{int32_t(i), w, a, std::min(len[w], a + bs)});
      }
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t bi = 0; bi < int64_t(blks.size()); ++bi) {
      const Blk bk = blks[size_t(bi)];
      const size_t i = size_t(bk.task);
      const Out& o = outs[i];
      if (bk.what == 0) {
        std::copy(o.terms.begin() + bk.a, o.terms.begin() + bk.e,
                  P.mat_terms.begin() + b_terms[i] + bk.a);
      } else if (bk.what == 1) {
        for (int64_t r = bk.a; r < bk.e; ++r) {
          TRec x = o.recs[size_t(r)];
          x.mat += int32_t(b_terms[i]);
          recs[size_t(b_recs[i] + r)] = x;
        }
      } else if (bk.what == 2) {
        for (int64_t g = bk.a; g < bk.e; ++g) {
          const GRef ref = o.tile_groups[size_t(g)];
          Group gr = outs[ref.first].groups[ref.second];
          gr.t_begin += int32_t(b_terms[ref.first]);
          gr.t_end += int32_t(b_terms[ref.first]);
          P.mat_groups[size_t(b_tg[i] + g)] = gr;
        }
      } else {
        for (int64_t l = bk.a; l < bk.e; ++l) {
          hx::OutLeaf L = o.leaves[size_t(l)];
          const int64_t wb = L.kind == 1 ? b_far[i] : b_near[i];
          L.ws_off += wb;
          for (int32_t k = L.tile_begin; k < L.tile_end; ++k) {
            Tile tl = o.tiles[k];
            tl.out_off += wb;
            tl.g_begin += int32_t(b_tg[i]);
            tl.g_end += int32_t(b_tg[i]);
            tl.aux += int32_t(b_sumsq[i]);
            P.mat_tiles[size_t(b_tiles[i]) + k] = tl;
          }
          L.tile_begin += int32_t(b_tiles[i]);
          L.tile_end += int32_t(b_tiles[i]);
          L.sumsq_begin += int32_t(b_sumsq[i]);
          L.sumsq_end += int32_t(b_sumsq[i]);
          if (L.implicit || L.troot >= 0) {
            L.g_begin += int32_t(b_tg[i]);
            L.g_end += int32_t(b_tg[i]);
          }
          if (L.troot >= 0) L.troot += int32_t(b_nodes[i]);
          for (int32_t k = L.tsub_begin; k < L.tsub_end; ++k) {
            hx::TSubBlock tb = o.tsub[size_t(k)];
            tb.off += wb;
            P.tsub[size_t(b_tsub[i]) + size_t(k)] = tb;
          }
          L.tsub_begin += int32_t(b_tsub[i]);
          L.tsub_end += int32_t(b_tsub[i]);
          P.leaves[size_t(b_leaves[i] + l)] = L;
        }
      }
    }
    lap("merge copy");
    if (!P.tsub.empty()) P.needs_eye = true;  // the iterative route applies T_sub blocks as T_b I
    if (b_nodes[no] > 0) {  // traditional-mode conversion trees
      P.tnodes.resize(size_t(b_nodes[no]));
      P.tkids.resize(size_t(b_kids[no]));
      for (size_t i = 0; i < no; ++i) {
        const Out& o = outs[i];
        for (size_t k = 0; k < o.tnodes.size(); ++k) {
          hx::TNode x = o.tnodes[k];
          if (x.term >= 0) x.term += int32_t(b_terms[i]);
          x.kid_begin += int32_t(b_kids[i]);
          x.kid_end += int32_t(b_kids[i]);
          P.tnodes[size_t(b_nodes[i]) + k] = x;
        }
        for (size_t k = 0; k < o.tkids.size(); ++k)
          P.tkids[size_t(b_kids[i]) + k] = o.tkids[k] + int32_t(b_nodes[i]);
        P.trad_matvecs += o.trad_cols;
      }
    }
    // restrict log in the reference's visiting order: each subtree's log goes right after
    // the top-part entries logged before the subtree was deferred
    if (logging) {
      const Out& top = outs[0];
      size_t pos = 0;
      auto append = [&](const Out& o, size_t a, size_t e) {
        P.log_block.insert(P.log_block.end(), o.log_block.begin() + a, o.log_block.begin() + e);
        P.log_kind.insert(P.log_kind.end(), o.log_kind.begin() + a, o.log_kind.begin() + e);
        P.log_a.insert(P.log_a.end(), o.log_a.begin() + a, o.log_a.begin() + e);
        P.log_b.insert(P.log_b.end(), o.log_b.begin() + a, o.log_b.begin() + e);
        P.log_rank.insert(P.log_rank.end(), o.log_rank.begin() + a, o.log_rank.begin() + e);
      };
      for (size_t i = 1; i < no; ++i) {
        const size_t at = size_t(task_log_pos[i - 1]);
        append(top, pos, at);
        pos = at;
        append(outs[i], 0, outs[i].log_block.size());
      }
      append(top, pos, top.log_block.size());
    }
    lap("merge log");
    hx_plan_info& I = P.info;
    for (const Out& o : outs) {
      I.n_terms_real += o.n_terms_real;
      I.n_terms_expand += o.n_terms_expand + o.n_mixed;
      I.n_dxd += o.n_dxd;
      for (int k = 0; k < 3; ++k) I.created[k] += o.created[k];
      I.n_far += o.n_far;
      I.n_near += o.n_near;
      I.max_out_dim = std::max(I.max_out_dim, o.max_out_dim);
      I.flops_near += o.flops_near;
      I.bytes_near += o.bytes_near;
    }
  }

  int64_t ws_far_total = 0, ws_near_total = 0;
  std::vector<int64_t> task_log_pos;
  std::vector<int32_t> order;  // terms sorted by X-group
  std::vector<int64_t> trans_off;  // per A node: offset of its transposed copy (or -1)

  // --------------------------------------------------------------- grouped term factors
  // workspace bound (doubles) for one batch of gathered factors, and for its cores
  static constexpr int64_t budget = int64_t(1) << 28;

  struct GInfo {
    int32_t b0, b1;   // term range in `order`
    int32_t X, rows_cl, rho;
    int8_t side;
    int64_t R, kr, ktot;
    std::vector<int> leaves;  // leaves of X (DFS order)
    int64_t srows;            // rows of the stacked cores (sum of the leaf ranks)
    int64_t n_core_tiles, n_core_groups, n_core_terms;
    int64_t n_fac_tiles, n_fac_groups, n_fac_terms;
    double mv, bytes;
    // offsets (second pass)
    int64_t out, gat, core;
    int64_t o_gather, o_ct, o_cg, o_cm, o_ft, o_fg, o_fm;
  };
  std::vector<GInfo> G;

  // Stacked-core layout of one X-group.  The low-rank leaves of X are ordered by their
  // middle cluster (sigma_l on the A side, tau_l on the B side) and then by output rows;
  // consecutive leaves sharing the middle cluster whose middle factors are adjacent in the
  // pool (the panel layout of hx_assemble / pack_operand) form one run = one term
  // [V_l1 .. V_lp]^T G[mid] of Sum k rows, so a 64-row core tile is filled by one panel
  // instead of one 10-50-row leaf.  `idx` holds positions in g.leaves; soff[i] is the
  // first stacked row of leaf g.leaves[i].
  struct CoreRun {
    int32_t first, count;  // range in idx
    int64_t row, rows;     // stacked rows
  };
  void core_layout(const GInfo& g, const hx_operand& opX, std::vector<int32_t>& idx,
                   std::vector<CoreRun>& runs, std::vector<int64_t>* soff) const {
    idx.clear();
    runs.clear();
    const int nl = int(g.leaves.size());
    for (int i = 0; i < nl; ++i) {
      const int l = g.leaves[size_t(i)];
      if (isF(opX, l) && opX.rank[l] > 0) idx.push_back(i);
    }
    auto mid = [&](int l) { return g.side == 0 ? t.sigma[l] : t.tau[l]; };
    auto outc = [&](int l) { return g.side == 0 ? t.tau[l] : t.sigma[l]; };
    auto midf = [&](int l) { return g.side == 0 ? opX.v_off[l] : opX.u_off[l]; };
    std::sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) {
      const int la = g.leaves[size_t(a)], lb = g.leaves[size_t(b)];
      const int ma = mid(la), mb = mid(lb);
      if (ma != mb) return ma < mb;
      return lo(outc(la)) < lo(outc(lb));
    });
    if (soff) soff->assign(size_t(nl), -1);
    int64_t row = 0;
    for (int32_t j = 0; j < int32_t(idx.size()); ++j) {
      const int l = g.leaves[size_t(idx[size_t(j)])];
      const int kl = opX.rank[l];
      bool ext = false;
      if (!runs.empty()) {
        const int p = g.leaves[size_t(idx[size_t(j - 1)])];
        ext = mid(p) == mid(l) && midf(l) == midf(p) + sz(mid(p)) * int64_t(opX.rank[p]);
      }
      if (ext) {
        runs.back().count++;
        runs.back().rows += kl;
      } else {
        // runs start on 8-row boundaries: a run's rows then fill whole 8 x 8 DMMA
        // fragments instead of sharing a fragment with the previous run's K range
        row = (row + core_align - 1) / core_align * core_align;
        runs.push_back(CoreRun{j, 1, row, kl});
      }
      if (soff) (*soff)[size_t(idx[size_t(j)])] = row;
      row += kl;
    }
  }

  static int64_t nbands(int64_t rows, int T) { return (rows + T - 1) / T; }
  static int64_t bands_hit(int64_t a, int64_t len, int64_t nb, int T) {
    const int64_t b0 = std::max<int64_t>(a / T, 0);
    const int64_t b1 = std::min<int64_t>((a + len - 1) / T, nb - 1);
    return b1 >= b0 ? b1 - b0 + 1 : 0;
  }

  // Tiles of an R x C output (ld R) whose row band i uses group gbase + i; gcol[jt]: first
  // column record of column tile jt (MODE_GCOL tiles read the X-group's virtual G).
  void write_band_tiles(Tile* tiles, uint8_t out_buf, int64_t out_off, int64_t R, int64_t C,
                        int64_t row_base, int32_t gbase, const int32_t* gcol) const {
    int64_t w = 0;
    for (int64_t i = 0, band = 0; i < R; i += T, ++band) {
      const int64_t r1 = std::min<int64_t>(R, i + T);
      for (int64_t j = 0; j < C; j += T) {
        Tile& tl = tiles[w++];
        std::memset(&tl, 0, sizeof(tl));
        tl.out_off = out_off + i + j * R;
        tl.out_ld = int32_t(R);
        tl.row0 = int32_t(row_base + i);
        tl.col0 = int32_t(j);
        tl.rows = int16_t(r1 - i);
        tl.cols = int16_t(std::min<int64_t>(C, j + T) - j);
        tl.g_begin = gbase + int32_t(band);
        tl.g_end = gbase + int32_t(band) + 1;
        tl.aux = gcol[j / T];
        tl.out_buf = out_buf;
        tl.mode = hx::MODE_GCOL;
      }
    }
  }

  bool verbose = std::getenv("HX_PLAN_VERBOSE") != nullptr;
  std::chrono::steady_clock::time_point tg0;
  void lap(const char* what) {
    if (!verbose) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hx plan]   %s %.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - tg0).count());
    tg0 = now;
  }

  void build_groups() {
    tg0 = std::chrono::steady_clock::now();
    const int nn = t.n_nodes;
    const size_t nr = recs.size();
    // counting sort of the terms by (side, X), over the keys that occur (a masked plan --
    // one chunk of 65 on config 4 -- touches a small part of the 2 n_nodes key space, and
    // per-thread histograms over all of it cost more than the sort itself)
    auto key = [&](const TRec& r) { return r.side * nn + (r.side == 0 ? r.pc : r.qc); };
    const int nk_all = 2 * nn;
    std::vector<uint8_t> used(size_t(nk_all), 0);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < int64_t(nr); ++i) used[size_t(key(recs[size_t(i)]))] = 1;
    std::vector<int32_t> kid(size_t(nk_all), -1), ckey;
    for (int k = 0; k < nk_all; ++k)
      if (used[size_t(k)]) {
        kid[size_t(k)] = int32_t(ckey.size());
        ckey.push_back(k);
      }
    const int nk = int(ckey.size());
    std::vector<int32_t> cnt(size_t(nk) + 1, 0);
    // parallel counting sort: per-thread histograms over contiguous slices of recs, then
    // (key, thread)-ordered offsets, so the order is the same as a sequential stable sort
    const int nth = std::max(1, std::min(omp_get_max_threads(), int(nr / 65536) + 1));
    std::vector<int32_t> hist(size_t(nth) * size_t(std::max(nk, 1)), 0);
    std::vector<int32_t> block_sum(size_t(nth), 0);
    order.resize(nr);
#pragma omp parallel num_threads(nth)
    {
      const int nth = omp_get_num_threads();  // the team actually granted
      const int th = omp_get_thread_num();
      const size_t a = nr * size_t(th) / size_t(nth), e = nr * size_t(th + 1) / size_t(nth);
      int32_t* h = &hist[size_t(th) * size_t(std::max(nk, 1))];
      for (size_t i = a; i < e; ++i) h[kid[size_t(key(recs[i]))]]++;
#pragma omp barrier
      // (key, thread)-ordered exclusive prefix, in parallel over key blocks
      const int kb0 = int(int64_t(nk) * th / nth), kb1 = int(int64_t(nk) * (th + 1) / nth);
      int32_t bsum = 0;
      for (int k = kb0; k < kb1; ++k)
        for (int q = 0; q < nth; ++q) bsum += hist[size_t(q) * size_t(nk) + size_t(k)];
      block_sum[size_t(th)] = bsum;
#pragma omp barrier
      int32_t run = 0;
      for (int q = 0; q < th; ++q) run += block_sum[size_t(q)];
      for (int k = kb0; k < kb1; ++k) {
        cnt[size_t(k)] = run;
        for (int q = 0; q < nth; ++q) {
          int32_t& x = hist[size_t(q) * size_t(nk) + size_t(k)];
          const int32_t c = x;
          x = run;
          run += c;
        }
      }
      if (th == nth - 1) cnt[size_t(nk)] = run;
#pragma omp barrier
      for (size_t i = a; i < e; ++i) order[size_t(h[kid[size_t(key(recs[i]))]]++)] = int32_t(i);
    }
    lap("order");
    G.clear();
    G.resize(size_t(nk));
#pragma omp parallel for schedule(static)
    for (int g = 0; g < nk; ++g) {
      GInfo& gi = G[size_t(g)];
      gi.b0 = cnt[size_t(g)];
      gi.b1 = cnt[size_t(g) + 1];
      gi.side = int8_t(ckey[size_t(g)] >= nn ? 1 : 0);
      gi.X = ckey[size_t(g)] - gi.side * nn;
    }
    const int64_t ng = int64_t(G.size());
    lap("sort");
    // pass 1 (parallel): leaves of X and work counts
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t gi_ = 0; gi_ < ng; ++gi_) {
      GInfo& g = G[gi_];
      const hx_operand& opX = g.side == 0 ? A : B;
      g.rows_cl = g.side == 0 ? t.tau[g.X] : t.sigma[g.X];
      g.rho = g.side == 0 ? t.sigma[g.X] : t.tau[g.X];
      g.R = sz(g.rows_cl);
      g.kr = sz(g.rho);
      g.ktot = 0;
      for (int32_t i = g.b0; i < g.b1; ++i) g.ktot += recs[order[i]].k;
      g.mv = 0;
      g.bytes = 0;
      subtree_leaves(opX, g.X, g.leaves, g.mv, g.bytes);
      const int64_t ct = nbands(g.ktot, T);
      const int64_t nb = nbands(g.R, T);
      g.n_fac_terms = 0;
      for (int l : g.leaves) {
        const int ol = g.side == 0 ? t.tau[l] : t.sigma[l];
        if (isF(opX, l) && opX.rank[l] == 0) continue;
        g.n_fac_terms += bands_hit(lo(ol) - lo(g.rows_cl), sz(ol), nb, T);
      }
      int64_t terms = 0;
      int64_t nbs = 0;
      {
        thread_local std::vector<int32_t> idx;
        thread_local std::vector<CoreRun> runs;
        core_layout(g, opX, idx, runs, nullptr);
        g.srows = runs.empty() ? 0 : runs.back().row + runs.back().rows;
        nbs = nbands(g.srows, T);
        for (const CoreRun& cr : runs) terms += bands_hit(cr.row, cr.rows, nbs, T);
      }
      g.n_core_terms = terms;
      g.n_core_groups = nbs;
      g.n_core_tiles = nbs * ct;
      g.n_fac_groups = nb;
      g.n_fac_tiles = nb * ct;
    }
    lap("pass1");
    // pass 2 (sequential): batches and offsets
    int64_t gat_cur = 0, core_cur = 0;
    int64_t o_gather = 0, o_ct = 0, o_cg = 0, o_cm = 0, o_ft = 0, o_fg = 0, o_fm = 0;
    auto close_batch = [&](int64_t gi_end) {
      hx_plan::Batch& b = P.batches.back();
      b.gather_end = o_gather;
      b.core_end = o_ct;
      b.fac_end = o_ft;
      b.cg_end = o_cg;
      b.cm_end = o_cm;
      b.fg_end = o_fg;
      b.fm_end = o_fm;
      b.g_end = gi_end;
    };
    auto open_batch = [&](int64_t gi_begin) {
      hx_plan::Batch b{};
      b.gather_begin = o_gather;
      b.core_begin = o_ct;
      b.fac_begin = o_ft;
      b.cg_begin = o_cg;
      b.cm_begin = o_cm;
      b.fg_begin = o_fg;
      b.fm_begin = o_fm;
      b.g_begin = gi_begin;
      P.batches.push_back(b);
    };
    open_batch(0);
    for (int64_t gi_ = 0; gi_ < ng; ++gi_) {
      GInfo& g = G[gi_];
      const int64_t gat_need = align16(g.kr * g.ktot);
      const int64_t core_need = align16(g.srows * g.ktot);
      // the thin factors are read in place (ColRec); gat_cur only bounds a batch's size
      if ((gat_cur + gat_need > budget || core_cur + core_need > budget) &&
          (gat_cur > 0 || core_cur > 0)) {
        close_batch(gi_);
        open_batch(gi_);
        gat_cur = core_cur = 0;
      }
      g.out = P.term_elems;
      P.term_elems = align16(P.term_elems + g.R * g.ktot);
      g.gat = gat_cur;
      gat_cur += gat_need;
      g.core = core_cur;
      core_cur += core_need;
      P.core_elems = std::max(P.core_elems, core_cur);
      g.o_gather = o_gather;
      o_gather += g.b1 - g.b0;
      g.o_ct = o_ct;
      o_ct += g.n_core_tiles;
      g.o_cg = o_cg;
      o_cg += g.n_core_groups;
      g.o_cm = o_cm;
      o_cm += g.n_core_terms;
      g.o_ft = o_ft;
      o_ft += g.n_fac_tiles;
      g.o_fg = o_fg;
      o_fg += g.n_fac_groups;
      g.o_fm = o_fm;
      o_fm += g.n_fac_terms;
      P.info.flops_form += double(g.ktot) * g.mv;
      P.info.bytes_form += double(g.b1 - g.b0) * g.bytes + 8.0 * double(g.ktot) * double(g.kr + g.R);
      P.info.n_xgroups++;
    }
    close_batch(ng);
    P.gcols.resize(size_t(o_gather));
    P.core_tiles.resize(size_t(o_ct));
    P.core_groups.resize(size_t(o_cg));
    P.core_terms.resize(size_t(o_cm));
    P.fac_tiles.resize(size_t(o_ft));
    P.fac_groups.resize(size_t(o_fg));
    P.fac_terms.resize(size_t(o_fm));
    lap("pass2");
    // transposed copies of the dense blocks of dense x H-block terms (ragged trees)
    trans_off.clear();
    for (const TRec& r : recs) {
      if (!r.dg) continue;
      P.needs_eye = true;
      if (r.side != 1) continue;
      if (trans_off.empty()) trans_off.assign(size_t(t.n_nodes), -1);
      if (trans_off[size_t(r.pc)] >= 0) continue;
      const int tp = t.tau[r.pc], rp = t.sigma[r.pc];
      trans_off[size_t(r.pc)] = P.dtrans_elems;
      P.dtrans.push_back(hx::TransRec{A.d_off[r.pc], P.dtrans_elems, int32_t(sz(tp)),
                                      int32_t(sz(rp))});
      P.dtrans_elems = align16(P.dtrans_elems + sz(tp) * sz(rp));
    }
    // pass 3 (parallel): column records of the virtual G and the computed-factor offsets of
    // the materialization terms -- everything the materialization launch needs
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t gi_ = 0; gi_ < ng; ++gi_) {
      const GInfo& g = G[gi_];
      // the thin factors side by side as columns of G; patch the materialization terms
      int64_t col = 0;
      for (int32_t i = g.b0; i < g.b1; ++i) {
        // the group's records and their materialization terms are scattered (creation
        // order): fetch a few ahead
        if (i + 8 < g.b1) {
          const TRec& rn = recs[order[i + 8]];
          __builtin_prefetch(&rn, 0, 1);
          if (i + 4 < g.b1) __builtin_prefetch(&P.mat_terms[recs[order[i + 4]].mat], 1, 1);
        }
        const TRec& r = recs[order[i]];
        hx::ColRec& cp = P.gcols[size_t(g.o_gather + (i - g.b0))];
        cp.buf = g.side == 0 ? hx::BUF_B : hx::BUF_A;
        cp.src_off = g.side == 0 ? B.u_off[r.qc] : A.v_off[r.pc];
        if (r.dg) {  // dense thin matrix: D_qc itself, or the transposed copy of D_pc
          if (g.side == 0) {
            cp.src_off = B.d_off[r.qc];
          } else {
            cp.buf = hx::BUF_GATHER;
            cp.src_off = trans_off[size_t(r.pc)];
          }
        }
        cp.col = int32_t(col);
        cp.k = r.k;
        cp.ld = int32_t(g.kr);
        Term& mt = P.mat_terms[r.mat];
        if (g.side == 0) {
          mt.a_off = g.out + col * g.R;
          mt.a_ld = int32_t(g.R);
        } else {
          mt.b_off = g.out + col * g.R;
          mt.b_ld = int32_t(g.R);
        }
        col += r.k;
      }
    }
    lap("pass3");
  }

  // pass 4 for one batch (parallel over its groups): stacked-core and X G work lists.
  // Deferred plans run this batch by batch inside hx_product, overlapping the device.
  void fill_batch(int64_t bi) {
    const hx_plan::Batch& bt = P.batches[size_t(bi)];
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t gi_ = bt.g_begin; gi_ < bt.g_end; ++gi_) {
      const GInfo& g = G[gi_];
      const hx_operand& opX = g.side == 0 ? A : B;
      const uint8_t xbuf = g.side == 0 ? hx::BUF_A : hx::BUF_B;
      const uint8_t gbuf = g.side == 0 ? hx::BUF_B : hx::BUF_A;  // the thin factors
      // first column record of every 64-column tile of G
      thread_local std::vector<int32_t> gcol;
      gcol.assign(size_t(nbands(g.ktot, T)), 0);
      {
        int32_t rec = int32_t(g.o_gather);
        for (size_t jt = 0; jt < gcol.size(); ++jt) {
          const int64_t j = int64_t(jt) * T;
          while (P.gcols[size_t(rec)].col + P.gcols[size_t(rec)].k <= j) ++rec;
          gcol[jt] = rec;
        }
      }
      // stacked cores S (srows x ktot, ld srows): rows [off_l, off_l + k_l) = V_l^T G[rho_l]
      // (A side) or U_l^T G[rho_l] (B side)
      const int64_t nbs = nbands(g.srows, T);
      const int64_t nb = nbands(g.R, T);
      thread_local std::vector<int32_t> idx;
      thread_local std::vector<CoreRun> runs;
      thread_local std::vector<int64_t> soff;
      core_layout(g, opX, idx, runs, &soff);
      {
        // runs ascend in stacked rows, so their (run, band) pieces come out band-sorted
        int64_t w = g.o_cm;
        int64_t band_next = 0;
        for (const CoreRun& cr : runs) {
          const int l = g.leaves[size_t(idx[size_t(cr.first)])];
          const int rl = g.side == 0 ? t.sigma[l] : t.tau[l];
          const int64_t roff = lo(rl) - lo(g.rho);
          const int64_t mid_f = g.side == 0 ? opX.v_off[l] : opX.u_off[l];
          const Term tm = make_term(xbuf, mid_f, int32_t(sz(rl)), 1, gbuf, roff,
                                    int32_t(g.kr), 2, int32_t(sz(rl)), cr.row, 0, cr.rows,
                                    g.ktot);
          for (int64_t band = cr.row / T; band <= (cr.row + cr.rows - 1) / T; ++band) {
            while (band_next <= band)
              P.core_groups[size_t(g.o_cg + band_next++)].t_begin = int32_t(w);
            P.core_terms[size_t(w++)] = tm;
          }
        }
        while (band_next < nbs) P.core_groups[size_t(g.o_cg + band_next++)].t_begin = int32_t(w);
        for (int64_t band = 0; band < nbs; ++band)
          P.core_groups[size_t(g.o_cg + band)].t_end =
              band + 1 < nbs ? P.core_groups[size_t(g.o_cg + band + 1)].t_begin : int32_t(w);
        write_band_tiles(&P.core_tiles[size_t(g.o_ct)], hx::BUF_CORE, g.core, g.srows, g.ktot, 0,
                         int32_t(g.o_cg), gcol.data());
      }
      // row bands of X G (A side) / X^T G (B side): count per band, then place (leaves in
      // DFS order within a band)
      {
        thread_local std::vector<int32_t> pos;
        pos.assign(size_t(nb) + 1, 0);
        const int nl = int(g.leaves.size());
        const int64_t base = lo(g.rows_cl);
        for (int i = 0; i < nl; ++i) {
          const int l = g.leaves[size_t(i)];
          if (isF(opX, l) && opX.rank[l] == 0) continue;
          const int ol = g.side == 0 ? t.tau[l] : t.sigma[l];
          for (int64_t band = (lo(ol) - base) / T; band <= (lo(ol) + sz(ol) - 1 - base) / T;
               ++band)
            pos[size_t(band) + 1]++;
        }
        for (int64_t band = 0; band < nb; ++band) {
          pos[size_t(band) + 1] += pos[size_t(band)];
          P.fac_groups[size_t(g.o_fg + band)] =
              Group{int32_t(g.o_fm + pos[size_t(band)]), int32_t(g.o_fm + pos[size_t(band) + 1])};
        }
        // low-rank leaves first, then dense ones: on the B side their staging layouts
        // differ (U_l vs D_l^T), and a chunk of the GEMM holds one layout, so interleaving
        // them in DFS order would cut the band's K stream into short chunks
        for (int pass = 0; pass < 2; ++pass)
        for (int i = 0; i < nl; ++i) {
          const int l = g.leaves[size_t(i)];
          const int rl = g.side == 0 ? t.sigma[l] : t.tau[l];  // middle-cluster part
          const int ol = g.side == 0 ? t.tau[l] : t.sigma[l];  // output rows
          const bool lr = isF(opX, l);
          if (lr != (pass == 0)) continue;
          const int kl = lr ? opX.rank[l] : 0;
          if (lr && kl == 0) continue;
          const int64_t roff = lo(rl) - lo(g.rho);
          Term tm;
          if (lr) {
            const int64_t out_f = g.side == 0 ? opX.u_off[l] : opX.v_off[l];
            tm = make_term(xbuf, out_f, int32_t(sz(ol)), 0, hx::BUF_CORE,
                           g.core + soff[size_t(i)], int32_t(g.srows), 1, kl, lo(ol), 0, sz(ol),
                           g.ktot);
          } else {
            tm = make_term(xbuf, opX.d_off[l], int32_t(sz(t.tau[l])),
                           uint8_t(g.side == 0 ? 0 : 1), gbuf, roff, int32_t(g.kr), 2,
                           int32_t(sz(rl)), lo(ol), 0, sz(ol), g.ktot);
          }
          for (int64_t band = (lo(ol) - base) / T; band <= (lo(ol) + sz(ol) - 1 - base) / T;
               ++band)
            P.fac_terms[size_t(g.o_fm + pos[size_t(band)]++)] = tm;
        }
        write_band_tiles(&P.fac_tiles[size_t(g.o_ft)], hx::BUF_TERM, g.out, g.R, g.ktot,
                         lo(g.rows_cl), int32_t(g.o_fg), gcol.data());
      }
    }
  }

  // near blocks go after the far ones so the result download is two contiguous copies
  void place_near() {
    P.near_ws_begin = ws_far_total;
    P.tile_elems = ws_far_total + ws_near_total;
    for (hx::OutLeaf& L : P.leaves) {
      if (L.kind != 2) continue;
      L.ws_off += ws_far_total;
      for (int32_t i = L.tile_begin; i < L.tile_end; ++i) P.mat_tiles[i].out_off += ws_far_total;
    }
  }

  void run() {
    const auto t0 = std::chrono::steady_clock::now();
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
    std::vector<Out> outs(1);
    if (t.kind[0] != INNER) {
      // the root itself is a leaf: S(root) = {(A_root, B_root)} evaluated directly
      if (owned_sub[0]) {
        Walk w{outs[0], 0, {}, 0};
        const int tc = t.tau[0], sc = t.sigma[0];
        if (t.kind[0] == FAR) throw hx::Unsupported("admissible root block");
        create_dxd(w, tc, sc, 0, 0);
        outs[0].groups.push_back(Group{0, int32_t(outs[0].terms.size())});
        w.path.push_back(GRef{0, 0});
        const double m = double(sz(tc));
        const double fdd = 2.0 * m * m * m, edd = 2.0 * m * m;
        outs[0].flops_near += fdd;
        outs[0].bytes_near += 8.0 * (edd + m * m);
        outs[0].n_near++;
        std::vector<VGroup> vg;
        emit_leaf_tiles(w, 0, false, vg, 0, fdd, edd, {});
      }
    } else {
      std::vector<Task> tasks;
      {
        Walk w{outs[0], 0, {}, 0};
        const PairList root{{0, 0}};
        visit(w, 0, 0, root, choose_cut(), &tasks);
      }
      outs.resize(1 + tasks.size());
      for (const Task& tk : tasks) task_log_pos.push_back(tk.log_pos);
      std::vector<std::string> errors(tasks.size());
#pragma omp parallel for schedule(dynamic, 1)
      for (int64_t i = 0; i < int64_t(tasks.size()); ++i) {
        try {
          Walk w{outs[size_t(i) + 1], int32_t(i + 1), tasks[size_t(i)].path,
                 tasks[size_t(i)].path_K};
          int lvl = 0;
          visit(w, tasks[size_t(i)].c, lvl, tasks[size_t(i)].pend, 1 << 30, nullptr);
        } catch (const std::exception& e) {
          errors[size_t(i)] = e.what();
        }
      }
      for (const std::string& e : errors)
        if (!e.empty()) throw hx::Unsupported(e);
      if (std::getenv("HX_PLAN_VERBOSE"))
        std::fprintf(stderr, "[hx plan] %zu descent tasks, %.1f ms\n", tasks.size(),
                     std::chrono::duration<double, std::milli>(
                         std::chrono::steady_clock::now() - t0).count());
    }
    const auto tm0 = std::chrono::steady_clock::now();
    merge(outs);
    const auto tm1 = std::chrono::steady_clock::now();
    outs.clear();
    const auto t1 = std::chrono::steady_clock::now();
    if (std::getenv("HX_PLAN_VERBOSE"))
      std::fprintf(stderr, "[hx plan] merge %.1f ms, free %.1f ms\n",
                   std::chrono::duration<double, std::milli>(tm1 - tm0).count(),
                   std::chrono::duration<double, std::milli>(t1 - tm1).count());
    build_groups();
    const auto t2 = std::chrono::steady_clock::now();
    place_near();
    if (std::getenv("HX_PLAN_VERBOSE"))
      std::fprintf(stderr, "[hx plan] descent %.1f ms, groups %.1f ms, %zu terms\n",
                   std::chrono::duration<double, std::milli>(t1 - t0).count(),
                   std::chrono::duration<double, std::milli>(t2 - t1).count(), recs.size());
  }
};

}  // namespace

extern "C" int hx_plan_create(const hx_tree* tree, const hx_operand* a, const hx_operand* b,
                              const uint8_t* leaf_mask, int tile, int flags, hx_plan** out) {
  struct Range {  // NVTX range over the planning (no-op without a tool attached)
    Range() { nvtxRangePushA("hx::plan"); }
    ~Range() { nvtxRangePop(); }
  } range;
  return hx::guarded([&]() -> int {
    if (!tree || !a || !b || !out) return hx::fail(HX_EINVAL, "null argument");
    if (tile != 32 && tile != 64) return hx::fail(HX_EINVAL, "tile must be 32 or 64");
    if (tree->n_nodes <= 0 || tree->n_clusters <= 0) return hx::fail(HX_EINVAL, "empty tree");
    auto* plan = new hx_plan();
    std::memset(&plan->info, 0, sizeof(plan->info));
    plan->tile = tile;
    plan->tree = *tree;
    plan->opa = *a;
    plan->opb = *b;
    try {
      auto bld = std::make_shared<Builder>(plan->tree, plan->opa, plan->opb, leaf_mask, tile,
                                           *plan);
      bld->logging = (flags & HX_PLAN_LOG) != 0;
      bld->trad = (flags >> HX_PLAN_TRAD_SHIFT) & 3;
      plan->trad = bld->trad;
      const int ish = (flags >> HX_PLAN_IMPLICIT_SHIFT) & 31;
      bld->implicit_min = ish ? (int64_t(1) << ish) : 0;
      plan->logged = bld->logging;
      bld->run();
      Builder* raw = bld.get();
      plan->builder = bld;
      plan->fill_batch = [raw](int64_t i) { raw->fill_batch(i); };
      plan->batch_ready.assign(plan->batches.size(), 0);
      if (!(flags & HX_PLAN_DEFER)) hx::plan_fill_all(plan);
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
    I.gather_jobs = int64_t(plan->gcols.size());
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
  if (!plan->logged) return hx::fail(HX_EINVAL, "plan created without HX_PLAN_LOG");
  if (block) std::copy(plan->log_block.begin(), plan->log_block.end(), block);
  if (kind) std::copy(plan->log_kind.begin(), plan->log_kind.end(), kind);
  if (a_node) std::copy(plan->log_a.begin(), plan->log_a.end(), a_node);
  if (b_node) std::copy(plan->log_b.begin(), plan->log_b.end(), b_node);
  if (rank) std::copy(plan->log_rank.begin(), plan->log_rank.end(), rank);
  return HX_OK;
}

extern "C" void hx_plan_free(hx_plan* plan) { delete plan; }

namespace hx {
void plan_fill_all(hx_plan* plan) {
  for (size_t i = 0; i < plan->batches.size(); ++i)
    if (!plan->batch_ready[i]) {
      plan->fill_batch(int64_t(i));
      plan->batch_ready[i] = 1;
    }
}
}  // namespace hx

extern "C" int hx_plan_mma_flops(hx_plan* plan, double* flops) {
  if (!plan || !flops) return hx::fail(HX_EINVAL, "null argument");
  hx::plan_fill_all(plan);
  const hx::hvec<Tile>* tiles[3] = {&plan->core_tiles, &plan->fac_tiles, &plan->mat_tiles};
  const hx::hvec<Group>* groups[3] = {&plan->core_groups, &plan->fac_groups,
                                      &plan->mat_groups};
  const hx::hvec<Term>* terms[3] = {&plan->core_terms, &plan->fac_terms, &plan->mat_terms};
  const double tt = double(plan->tile) * plan->tile;
  for (int b = 0; b < 3; ++b) {
    double f = 0, u = 0;
    for (const Tile& tl : *tiles[b])
      for (int32_t g = tl.g_begin; g < tl.g_end; ++g) {
        const Group gr = (*groups[b])[g];
        for (int32_t i = gr.t_begin; i < gr.t_end; ++i) {
          const Term& tm = (*terms[b])[i];
          f += 2.0 * tt * double((tm.k + 3) & ~3);
          const int r0 = std::max(tl.row0, tm.r_lo), r1 = std::min(tl.row0 + tl.rows,
                                                                   tm.r_lo + tm.rows);
          const int c0 = std::max(tl.col0, tm.c_lo), c1 = std::min(tl.col0 + tl.cols,
                                                                   tm.c_lo + tm.cols);
          if (r1 > r0 && c1 > c0) u += 2.0 * double(r1 - r0) * double(c1 - c0) * tm.k;
        }
      }
    flops[b] = f;
    flops[3 + b] = u;
  }
  return HX_OK;
}

int64_t hx::panel_layout(const hx_tree* tree, const int8_t* payload, const int32_t* rank,
                         int64_t* u_off, int64_t* v_off, int64_t* d_off) {
  const int nn = tree->n_nodes;
  auto lo = [&](int cl) { return tree->c_lo[cl]; };
  auto sz = [&](int cl) { return tree->c_hi[cl] - tree->c_lo[cl]; };
  std::vector<int> lr, dn;
  for (int b = 0; b < nn; ++b) {
    if (tree->kind[b] == 0) continue;
    u_off[b] = v_off[b] = d_off[b] = 0;
    (payload[b] == 1 ? lr : dn).push_back(b);
  }
  int64_t pos = 0;
  // one factor region: leaves sorted by (panel cluster, start of the other cluster)
  auto region = [&](const int32_t* panel, const int32_t* other, int64_t* off) {
    std::vector<int> o(lr);
    std::sort(o.begin(), o.end(), [&](int a, int b) {
      if (panel[a] != panel[b]) return panel[a] < panel[b];
      return lo(other[a]) < lo(other[b]);
    });
    for (size_t i = 0; i < o.size(); ++i) {
      const int b = o[i];
      off[b] = pos;
      pos += sz(panel[b]) * int64_t(rank[b]);
      if (i + 1 == o.size() || panel[o[i + 1]] != panel[b]) pos = align16(pos);
    }
  };
  region(tree->tau, tree->sigma, u_off);
  region(tree->sigma, tree->tau, v_off);
  for (int b : dn) {
    d_off[b] = pos;
    pos = align16(pos + sz(tree->tau[b]) * sz(tree->sigma[b]));
  }
  return pos;
}

extern "C" int hx_operand_layout(const hx_tree* tree, const int8_t* payload, const int32_t* rank,
                                 int64_t* u_off, int64_t* v_off, int64_t* d_off,
                                 int64_t* pool_elems) {
  if (!tree || !payload || !rank || !u_off || !v_off || !d_off || !pool_elems)
    return hx::fail(HX_EINVAL, "null argument");
  return hx::guarded([&]() -> int {
    *pool_elems = hx::panel_layout(tree, payload, rank, u_off, v_off, d_off);
    return HX_OK;
  });
}

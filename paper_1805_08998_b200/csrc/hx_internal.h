// Host-side internals shared by the plan builder and the CUDA runtime (not part of the ABI).
#pragma once
#include <cstdint>
#include <cstdio>
#include <functional>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hx.h"
#include "hx_types.h"

namespace hx {

// std::vector whose resize() leaves POD elements uninitialized (the plan arrays are
// filled right after sizing; zeroing hundreds of MB first would double the memory traffic)
template <class T>
struct DefaultInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind {
    using other = DefaultInitAlloc<U>;
  };
  using std::allocator<T>::allocator;
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
};
template <class T>
using pvec = std::vector<T, DefaultInitAlloc<T>>;

// Page-locked host memory with a reuse cache (runtime.cu; errors.cpp carries a plain
// malloc fallback for planner-only builds).  The plan's device work lists live here so
// their uploads are true async DMA that overlaps planning of the next batch.
void* pinned_alloc(size_t bytes);
void pinned_free(void* p, size_t bytes);

template <class T>
struct PinnedAlloc {
  using value_type = T;
  PinnedAlloc() = default;
  template <class U>
  PinnedAlloc(const PinnedAlloc<U>&) {}
  T* allocate(size_t n) { return static_cast<T*>(pinned_alloc(n * sizeof(T))); }
  void deallocate(T* p, size_t n) { pinned_free(p, n * sizeof(T)); }
  template <class U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
  template <class U>
  bool operator==(const PinnedAlloc<U>&) const {
    return true;
  }
  template <class U>
  bool operator!=(const PinnedAlloc<U>&) const {
    return false;
  }
};
template <class T>
using hvec = std::vector<T, PinnedAlloc<T>>;

struct Unsupported : std::runtime_error {
  explicit Unsupported(const std::string& s) : std::runtime_error(s) {}
};
struct CudaFailure : std::runtime_error {
  explicit CudaFailure(const std::string& s) : std::runtime_error(s) {}
};
struct OutOfMemory : std::runtime_error {
  explicit OutOfMemory(const std::string& s) : std::runtime_error(s) {}
};

struct OutLeaf {
  int32_t id;
  int8_t kind;   // 1 far, 2 near
  int32_t m, n;
  int64_t row0, col0;
  int64_t ws_off;
  int32_t tile_begin, tile_end;
  int32_t sumsq_begin, sumsq_end;
  int64_t K;
  double fdd, edd;
  // implicit route (far leaves with min(m, n) >= the plan's threshold): no tiles and no
  // workspace; the leaf's terms are the groups [g_begin, g_end) of mat_groups
  int8_t implicit;
  int32_t g_begin, g_end;
  // implicit route: the leaf's materialized part T_sub is block-sparse, the dense blocks
  // [tsub_begin, tsub_end) of hx_plan::tsub (none: everything is sketched)
  int32_t tsub_begin, tsub_end;
  // traditional mode (hmult_traditional): root of the leaf's fold tree in hx_plan::tnodes
  // (-1 otherwise); the path groups [g_begin, g_end) hold its inherited low-rank terms
  int32_t troot;
};

// One dense block of an implicit leaf's T_sub: the small sub-block terms of the leaf that
// are materialized rather than sketched, gathered by their outermost small virtual block
// (h x w, column-major at BUF_TILE + off, ld h; global coordinates r0, c0).
struct TSubBlock {
  int64_t off;
  int64_t r0, c0;
  int32_t h, w;
};

// Traditional-mode conversion tree of a far leaf (multiply.py:140-263).  Items name one
// term of mat_terms on the node's block; folds combine their children by pairwise
// truncated summation (fast_truncate_sum, lowrank.py:123-138); a stack truncates the
// concatenation of its children once (a compressor converter on the pair product).
enum TKind : int8_t { TN_LR = 0, TN_DD = 1, TN_FOLD = 2, TN_STACK = 3 };
struct TNode {
  int8_t kind;
  int8_t sort;      // leaf root: children in decreasing-norm order (multiply.py:222-224)
  int32_t term;     // items: index into mat_terms
  int32_t m, n;
  int64_t row0, col0;
  int32_t kid_begin, kid_end;  // children: hx_plan::tkids[kid_begin, kid_end)
};

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
void plan_fill_all(hx_plan* plan);

// Operand pool offsets in panel order (payload and rank given): left factors grouped by
// row cluster (ascending column start), right factors by column cluster (ascending row
// start), then dense leaves; 16-element padding only at panel ends, so the factors of a
// block row / column panel form one column-major matrix.  Returns the pool size.
int64_t panel_layout(const hx_tree* tree, const int8_t* payload, const int32_t* rank,
                     int64_t* u_off, int64_t* v_off, int64_t* d_off);

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const Unsupported& e) {
    return fail(HX_EUNSUPPORTED, e.what());
  } catch (const CudaFailure& e) {
    return fail(HX_ECUDA, e.what());
  } catch (const OutOfMemory& e) {
    return fail(HX_ENOMEM, e.what());
  } catch (const std::bad_alloc&) {
    return fail(HX_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(HX_EINVAL, e.what());
  }
}

}  // namespace hx

struct hx_plan {
  int tile = 64;
  hx::hvec<hx::Term> core_terms, fac_terms, mat_terms;
  hx::hvec<hx::Tile> core_tiles, fac_tiles, mat_tiles;
  hx::hvec<hx::Group> core_groups, fac_groups, mat_groups;
  std::vector<hx::Group> mat_groups_all;  // one per creation block (real or virtual)
  hx::pvec<hx::OutLeaf> leaves;
  hx::pvec<hx::TSubBlock> tsub;  // T_sub blocks of the implicit leaves
  int64_t core_elems = 0, term_elems = 0, tile_elems = 0, gather_elems = 0;
  hx::hvec<hx::ColRec> gcols;  // thin factors of each X-group (virtual G)
  std::vector<hx::TransRec> dtrans;  // transposed dense blocks (dense x H-block terms)
  int64_t dtrans_elems = 0;
  bool needs_eye = false;            // some term uses the identity operand (BUF_EYE)
  // X-groups are processed in batches whose gathered factors and cores fit a bounded
  // workspace (BUF_GATHER / BUF_CORE offsets restart at 0 in every batch)
  struct Batch {
    int64_t gather_begin, gather_end;
    int64_t core_begin, core_end;   // core tiles
    int64_t fac_begin, fac_end;     // fac tiles
    int64_t cg_begin, cg_end, cm_begin, cm_end;  // core groups / terms
    int64_t fg_begin, fg_end, fm_begin, fm_end;  // fac groups / terms
    int64_t g_begin, g_end;         // X-groups of the batch
  };
  std::vector<Batch> batches;
  // deferred plans (hx_plan_create with HX_PLAN_DEFER): the per-batch core / X G work
  // lists are filled by hx_product while the device runs earlier batches
  std::function<void(int64_t)> fill_batch;
  std::vector<uint8_t> batch_ready;
  std::shared_ptr<void> builder;
  hx_tree tree;           // copies of the caller's descriptors (arrays stay caller-owned)
  hx_operand opa, opb;
  int64_t near_ws_begin = 0;  // near-leaf blocks sit after all far blocks in BUF_TILE
  int32_t n_sumsq = 0;
  std::vector<int32_t> log_block, log_a, log_b, log_rank;
  bool logged = false;
  std::vector<int8_t> log_kind;
  // traditional mode: 0 off, 1 hierarchical pair conversion, 2 one truncation per pair
  int trad = 0;
  std::vector<hx::TNode> tnodes;
  std::vector<int32_t> tkids;
  int64_t trad_matvecs = 0;  // pending pairs converted (matvec count of a compressor converter)
  hx_plan_info info;
};

// Device runtime of the H x H product: context, pools, the product pipeline, results.
//
// hx_product replaces _multiply (/root/reference/pkg/src/hmat/multiply.py:207-249):
//   1. term formation  (cores, pushed-through factors)       grouped DMMA GEMM x 2
//   2. materialization of every output leaf from its terms   grouped DMMA GEMM x 1
//      (near leaves are final here: evaluate_dense, sumexpr.py:165-170)
//   3. recompression of far leaves to the requested policy (compress, compressors.py:441)
//      sketch  Y = T Omega -> Householder QR -> Bt = T^T Q -> QR -> Jacobi SVD of R
//      -> select_rank with the exact unsampled tail -> factors (U S, V)
//      blocks whose selected rank leaves less than `oversample` spare sketch columns are
//      redone with a doubled sketch; a sketch that spans the block is exact.
#include <sched.h>

#include <chrono>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_set>
#include <string>
#include <exception>
#include <functional>
#include <thread>
#include <vector>

#include "dense_la.cuh"
#include "dense_la_warp.cuh"
#include "gather_gemm.cuh"
#include "gemm.cuh"
#include "gemm_ws.cuh"
#include "iterative.cuh"
#include "qr_rows.cuh"
#include "traditional.cuh"
#include "hx_internal.h"

using namespace hx;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      throw hx::CudaFailure(std::string(#x) + ": " + cudaGetErrorString(e_));          \
  } while (0)

namespace {

constexpr int SMEM_CAP = 200 * 1024;  // dynamic shared memory per CTA we allow ourselves

template <class T>
struct DArr {
  T* p = nullptr;
  size_t cap = 0;
  void ensure(size_t n) {
    if (n <= cap && p) return;
    // growing: 25% slack (at most 2 GB) against regrowth by the next chunk or round
    const size_t grown = cap ? cap + std::min(cap / 4, (size_t(2) << 30) / sizeof(T)) : 0;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(n, 1);
    const size_t ask = std::max(want, grown);
    if (ask > want && cudaMalloc(&p, ask * sizeof(T)) == cudaSuccess) {
      cap = ask;
      return;
    }
    cudaGetLastError();
    if (cudaMalloc(&p, want * sizeof(T)) != cudaSuccess) {
      cudaGetLastError();
      throw hx::OutOfMemory("cudaMalloc of " + std::to_string(want * sizeof(T)) + " bytes");
    }
    cap = want;
  }
  void upload(const T* h, size_t n, cudaStream_t s) {
    ensure(n);
    if (n) CK(cudaMemcpyAsync(p, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  template <class Alloc>
  void upload(const std::vector<T, Alloc>& v, cudaStream_t s) {
    upload(v.data(), v.size(), s);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

// Standard normal test matrix (Box-Muller on a counter-based hash of (seed, index)).
__global__ void omega_kernel(double* om, int64_t n, uint64_t seed) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint64_t h1 = mix64(seed * 0x9E3779B97F4A7C15ULL + 2 * uint64_t(i) + 1);
  const uint64_t h2 = mix64(h1 ^ 0xD1B54A32D192ED03ULL);
  const double u1 = (double(h1 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  const double u2 = double(h2 >> 11) * (1.0 / 9007199254740992.0);
  om[i] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

__global__ void transpose_kernel(const TransRec* __restrict__ recs, const double* __restrict__ a,
                                 double* __restrict__ g) {
  const TransRec r = recs[blockIdx.x];
  const int64_t n = int64_t(r.rows) * r.cols;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    const int64_t i = e % r.rows, j = e / r.rows;
    g[r.dst_off + j + i * r.cols] = a[r.src_off + e];
  }
}

__global__ void eye_kernel(double* __restrict__ m, int64_t n, int ld) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < n) m[e] = (e % ld == e / ld) ? 1.0 : 0.0;
}

cudaEvent_t g_epoch;
bool g_epoch_set = false;
std::chrono::steady_clock::time_point g_host_epoch;

// Host-side milestones of one hx_product (HX_TIMING, after hx_timeline_epoch): milliseconds
// since the epoch, printed on exit, next to the device marks of hx_product_stats.t_marks.
struct HostMarks {
  bool on = g_epoch_set && std::getenv("HX_TIMING") != nullptr;
  const void* who;
  std::vector<std::pair<const char*, double>> m;
  explicit HostMarks(const void* c) : who(c) { mark("entry"); }
  void mark(const char* what) {
    if (!on) return;
    m.emplace_back(what, std::chrono::duration<double, std::milli>(
                             std::chrono::steady_clock::now() - g_host_epoch).count());
  }
  ~HostMarks() {
    if (!on) return;
    mark("exit");
    std::string line = "[hx host] ";
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%p:", who);
    line += buf;
    for (auto& x : m) {
      std::snprintf(buf, sizeof(buf), " %s %.1f", x.first, x.second);
      line += buf;
    }
    std::fprintf(stderr, "%s\n", line.c_str());
  }
};

}  // namespace

extern "C" int hx_timeline_epoch(void) {
  return guarded([&]() -> int {
    if (!g_epoch_set) CK(cudaEventCreate(&g_epoch));
    g_epoch_set = true;
    CK(cudaEventRecord(g_epoch, 0));
    g_host_epoch = std::chrono::steady_clock::now();
    return HX_OK;
  });
}

// ---- page-locked host memory cache (plan work lists) ----------------------------------
namespace hx {
namespace pin_detail {
std::mutex g_pin_mu;
std::multimap<size_t, void*> g_pin_free;  // capacity -> block
size_t g_pin_cached = 0;
std::unordered_set<void*>& g_unpinned() {
  static std::unordered_set<void*> s;
  return s;
}
constexpr size_t PIN_MIN = size_t(1) << 20;        // below: ordinary heap
constexpr size_t PIN_CACHE_MAX = size_t(32) << 30;  // cached bytes kept for reuse (pinning GBs costs ~1 s)
size_t pin_cap(size_t bytes) {
  size_t c = PIN_MIN;
  while (c < bytes) c <<= 1;
  return c;
}
}  // namespace pin_detail
using namespace pin_detail;

void* pinned_alloc(size_t bytes) {
  if (bytes < PIN_MIN) {
    void* p = std::malloc(bytes ? bytes : 1);
    if (!p) throw std::bad_alloc();
    return p;
  }
  const size_t cap = pin_cap(bytes);
  {
    std::lock_guard<std::mutex> g(g_pin_mu);
    auto it = g_pin_free.find(cap);
    if (it != g_pin_free.end()) {
      void* p = it->second;
      g_pin_free.erase(it);
      g_pin_cached -= cap;
      return p;
    }
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, cap, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    p = std::malloc(cap);  // no device / driver: still correct, just pageable
    if (!p) throw std::bad_alloc();
    // remember it is not page-locked: tag by registering nothing; freed with free()
    std::lock_guard<std::mutex> g(g_pin_mu);
    g_unpinned().insert(p);
  }
  return p;
}

void pinned_free(void* p, size_t bytes) {
  if (!p) return;
  if (bytes < PIN_MIN) {
    std::free(p);
    return;
  }
  const size_t cap = pin_cap(bytes);
  std::lock_guard<std::mutex> g(g_pin_mu);
  if (g_unpinned().erase(p)) {
    std::free(p);
    return;
  }
  if (g_pin_cached + cap <= PIN_CACHE_MAX) {
    g_pin_free.emplace(cap, p);
    g_pin_cached += cap;
  } else {
    cudaFreeHost(p);
  }
}
}  // namespace hx

// One term of an implicit-route leaf, clipped to the leaf (leaf-local row / column ranges).
struct ImplTerm {
  Term t;         // the materialization term (global coordinates, see hx_types.h)
  int lr;         // 1: factor pair (rows of Z / W gathered), 0: dense x dense (plain GEMM)
  int k;
  int ri, rn;     // leaf rows covered
  int ci, cn;     // leaf columns covered
  int64_t zrow;   // first row in the leaf's Z block (range pass)
  int64_t wrow;   // first row in the leaf's W block (co-range pass)
};

struct FarBlock {
  int leaf;        // index into plan leaves
  int m, n, mu;
  int64_t t_off;   // materialized block in BUF_TILE
  int l = 0;       // sketch width of the last round
  int dense = 0;   // 1: QR of T itself (m >= n, l == n)
  int rank = 0;
  int done = 0;
  int round = -1;
  int direct = 0;    // iterative route: output the produced factors (Y, Bt) as they are
  int degraded = 0;  // ACA ran out of rows without a certified zero
  // implicit route: terms and the row count of their stacked Z / W blocks
  int implicit = 0;
  std::vector<ImplTerm> it;
  std::vector<int> zorder, worder;  // it indices by Z row (lr, column band) / W row (row band)
  int64_t zrows = 0;
  int64_t zoff = 0;  // Z / W block in BUF_CORE for this round
  // pointers into that round's workspace
  double *Y = nullptr, *Bt = nullptr, *R = nullptr, *W = nullptr, *V = nullptr, *sig = nullptr;
  double* C1 = nullptr;  // Q^T Y_probe (implicit route)
  double* fro2 = nullptr;
};

// Several grouped-GEMM batches built on the host and uploaded at once; batch i is the tile
// range [cuts[i], cuts[i + 1]).
struct GemmSet {
  std::vector<Term> terms;
  std::vector<Tile> tiles;
  std::vector<Group> groups;
  std::vector<size_t> cuts{0};
  int32_t group(const Term* t, size_t n) {
    const int32_t g = int32_t(groups.size());
    groups.push_back(Group{int32_t(terms.size()), int32_t(terms.size() + n)});
    terms.insert(terms.end(), t, t + n);
    return g;
  }
  // tiles over an R x C output (ld) whose terms use coordinates (row0 + i, col0 + j)
  void cover(int32_t g, uint8_t out_buf, int64_t out_off, int32_t ld, int R, int C, int row0,
             int col0, uint8_t mode = MODE_STORE, int32_t* aux = nullptr) {
    for (int j = 0; j < C; j += 64)
      for (int i = 0; i < R; i += 64) {
        Tile tl;
        std::memset(&tl, 0, sizeof(tl));
        tl.out_off = out_off + i + int64_t(j) * ld;
        tl.out_ld = ld;
        tl.row0 = row0 + i;
        tl.col0 = col0 + j;
        tl.rows = int16_t(std::min(64, R - i));
        tl.cols = int16_t(std::min(64, C - j));
        tl.g_begin = g;
        tl.g_end = g + 1;
        tl.aux = aux ? (*aux)++ : -1;
        tl.out_buf = out_buf;
        tl.mode = mode;
        tiles.push_back(tl);
      }
  }
  // Like cover() for a sum of terms that each meet only a band of output rows, [lo,
  // lo + len) (band (0, R): every row): each 64-row tile lists only the terms whose band
  // meets it, through group entries over runs of terms sharing a band (terms are stored
  // once, full-band ones first), instead of staging every term of the sum in every tile.
  // presorted: ts already come in band order (terms sharing a band adjacent); full-band
  // terms then form ordinary runs that meet every tile
  void cover_banded(const std::vector<Term>& ts, const std::vector<std::pair<int, int>>& band,
                    uint8_t out_buf, int64_t out_off, int32_t ld, int R, int C, int row0,
                    int col0, bool presorted = false) {
    std::vector<int> o(ts.size());
    for (size_t i = 0; i < o.size(); ++i) o[i] = int(i);
    auto full = [&](int i) {
      return !presorted && band[size_t(i)].first <= 0 && band[size_t(i)].second >= R;
    };
    if (!presorted) std::stable_sort(o.begin(), o.end(), [&](int a, int b) {
      const bool fa = full(a), fb = full(b);
      if (fa != fb) return fa;
      if (!fa && band[size_t(a)] != band[size_t(b)]) return band[size_t(a)] < band[size_t(b)];
      // one staging layout per chunk: keep equal layouts adjacent
      const int la = ts[size_t(a)].a_kc * 4 + ts[size_t(a)].b_kc;
      const int lb = ts[size_t(b)].a_kc * 4 + ts[size_t(b)].b_kc;
      return la < lb;
    });
    const int32_t t0 = int32_t(terms.size());
    int32_t nf = 0;
    struct Run {
      int lo, hi;
      int32_t b, e;
    };
    std::vector<Run> runs;
    for (int i : o) {
      const int32_t t = int32_t(terms.size());
      terms.push_back(ts[size_t(i)]);
      if (full(i)) {
        ++nf;
        continue;
      }
      const int lo = band[size_t(i)].first, hi = lo + band[size_t(i)].second;
      if (!runs.empty() && runs.back().lo == lo && runs.back().hi == hi)
        runs.back().e = t + 1;
      else
        runs.push_back(Run{lo, hi, t, t + 1});
    }
    // runs by row tile (CSR, run order kept): a scan of every run per tile is quadratic on
    // the tallest leaves (65536 rows: 1024 row tiles x 10^4 runs)
    const int nrt = (R + 63) / 64;
    std::vector<int32_t> rs(size_t(nrt) + 1, 0), rl;
    for (const Run& r : runs) {
      if (r.hi <= r.lo) continue;
      const int a = std::max(0, r.lo / 64), b = std::min(nrt - 1, (r.hi - 1) / 64);
      for (int q = a; q <= b; ++q) rs[size_t(q) + 1]++;
    }
    for (int q = 0; q < nrt; ++q) rs[size_t(q) + 1] += rs[size_t(q)];
    rl.resize(size_t(rs[size_t(nrt)]));
    {
      std::vector<int32_t> fill(rs.begin(), rs.end() - 1);
      for (int32_t ri = 0; ri < int32_t(runs.size()); ++ri) {
        const Run& r = runs[size_t(ri)];
        if (r.hi <= r.lo) continue;
        const int a = std::max(0, r.lo / 64), b = std::min(nrt - 1, (r.hi - 1) / 64);
        for (int q = a; q <= b; ++q) rl[size_t(fill[size_t(q)]++)] = ri;
      }
    }
    for (int j = 0; j < C; j += 64)
      for (int i = 0; i < R; i += 64) {
        Tile tl;
        std::memset(&tl, 0, sizeof(tl));
        tl.out_off = out_off + i + int64_t(j) * ld;
        tl.out_ld = ld;
        tl.row0 = row0 + i;
        tl.col0 = col0 + j;
        tl.rows = int16_t(std::min(64, R - i));
        tl.cols = int16_t(std::min(64, C - j));
        tl.g_begin = int32_t(groups.size());
        if (nf) groups.push_back(Group{t0, t0 + nf});
        const int q = i / 64;
        for (int32_t x = rs[size_t(q)]; x < rs[size_t(q) + 1]; ++x) {
          const Run& r = runs[size_t(rl[size_t(x)])];
          groups.push_back(Group{r.b, r.e});
        }
        if (int32_t(groups.size()) == tl.g_begin) groups.push_back(Group{t0, t0});
        tl.g_end = int32_t(groups.size());
        tl.aux = -1;
        tl.out_buf = out_buf;
        tl.mode = MODE_STORE;
        tiles.push_back(tl);
      }
  }
  void cut() { cuts.push_back(tiles.size()); }
  size_t count(int b) const { return cuts[size_t(b) + 1] - cuts[size_t(b)]; }
};

struct GatherSet {
  std::vector<GTile> tiles;
  std::vector<GSeg> segs;
  std::vector<size_t> cuts{0};
  void cut() { cuts.push_back(tiles.size()); }
  size_t count(int b) const { return cuts[size_t(b) + 1] - cuts[size_t(b)]; }
};

// host threads this process may run on (the affinity mask: a GPU box slice can expose far
// fewer cores than std::thread::hardware_concurrency reports)
int host_threads() {
  static const int n = [] {
    if (const char* e = std::getenv("HX_LIST_THREADS")) return std::max(1, std::atoi(e));
    cpu_set_t set;
    CPU_ZERO(&set);
    if (sched_getaffinity(0, sizeof(set), &set) == 0) return std::max(1, int(CPU_COUNT(&set)));
    return std::max(1, int(std::thread::hardware_concurrency()));
  }();
  return n;
}

// fn(i) for i < n on host threads (contiguous ranges; the first exception is rethrown)
void par_for(int n, const std::function<void(int)>& fn) {
  const int hw = host_threads();
  const int nt = std::max(1, std::min(hw, n / 8));
  std::exception_ptr err;
  std::mutex em;
  auto run = [&](int t) {
    try {
      const int a0 = int(int64_t(n) * t / nt), a1 = int(int64_t(n) * (t + 1) / nt);
      for (int a = a0; a < a1; ++a) fn(a);
    } catch (...) {
      std::lock_guard<std::mutex> lk(em);
      err = std::current_exception();
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(run, t);
  run(0);
  for (auto& x : th) x.join();
  if (err) std::rethrow_exception(err);
}

// One batch of per-leaf work lists built by host threads over contiguous ranges of the
// active leaves, merged in leaf order: the same lists as a sequential build (body(i, gm,
// ga) appends leaf i's terms / tiles / gathered rows to the thread's own sets).
void par_build(const std::vector<int>& active, GemmSet& gm, GatherSet& ga,
               const std::function<void(int, GemmSet&, GatherSet&)>& body) {
  const int n = int(active.size());
  const int nt = std::max(1, std::min(host_threads(), n / 64));
  std::vector<GemmSet> gsets(static_cast<size_t>(nt));
  std::vector<GatherSet> asets(static_cast<size_t>(nt));
  auto run = [&](int t) {
    const int a0 = int(int64_t(n) * t / nt), a1 = int(int64_t(n) * (t + 1) / nt);
    for (int a = a0; a < a1; ++a) body(active[size_t(a)], gsets[size_t(t)], asets[size_t(t)]);
  };
  std::vector<std::thread> th;
  std::exception_ptr err;
  std::mutex em;
  for (int t = 1; t < nt; ++t)
    th.emplace_back([&, t] {
      try {
        run(t);
      } catch (...) {
        std::lock_guard<std::mutex> lk(em);
        err = std::current_exception();
      }
    });
  try {
    run(0);
  } catch (...) {
    std::lock_guard<std::mutex> lk(em);
    err = std::current_exception();
  }
  for (auto& x : th) x.join();
  if (err) std::rethrow_exception(err);
  // merge in leaf order, every thread copying its own sets to their final positions
  std::vector<size_t> o_t(size_t(nt) + 1), o_l(size_t(nt) + 1), o_g(size_t(nt) + 1),
      o_s(size_t(nt) + 1), o_x(size_t(nt) + 1);
  o_t[0] = gm.terms.size();
  o_l[0] = gm.tiles.size();
  o_g[0] = gm.groups.size();
  o_s[0] = ga.segs.size();
  o_x[0] = ga.tiles.size();
  for (int t = 0; t < nt; ++t) {
    o_t[size_t(t) + 1] = o_t[size_t(t)] + gsets[size_t(t)].terms.size();
    o_l[size_t(t) + 1] = o_l[size_t(t)] + gsets[size_t(t)].tiles.size();
    o_g[size_t(t) + 1] = o_g[size_t(t)] + gsets[size_t(t)].groups.size();
    o_s[size_t(t) + 1] = o_s[size_t(t)] + asets[size_t(t)].segs.size();
    o_x[size_t(t) + 1] = o_x[size_t(t)] + asets[size_t(t)].tiles.size();
  }
  gm.terms.resize(o_t[size_t(nt)]);
  gm.tiles.resize(o_l[size_t(nt)]);
  gm.groups.resize(o_g[size_t(nt)]);
  ga.segs.resize(o_s[size_t(nt)]);
  ga.tiles.resize(o_x[size_t(nt)]);
  auto merge = [&](int t) {
    const GemmSet& g = gsets[size_t(t)];
    const int32_t t0 = int32_t(o_t[size_t(t)]), g0 = int32_t(o_g[size_t(t)]);
    std::copy(g.terms.begin(), g.terms.end(), gm.terms.begin() + o_t[size_t(t)]);
    for (size_t k = 0; k < g.groups.size(); ++k)
      gm.groups[o_g[size_t(t)] + k] = Group{g.groups[k].t_begin + t0, g.groups[k].t_end + t0};
    for (size_t k = 0; k < g.tiles.size(); ++k) {
      Tile tl = g.tiles[k];
      tl.g_begin += g0;
      tl.g_end += g0;
      gm.tiles[o_l[size_t(t)] + k] = tl;
    }
    const GatherSet& x = asets[size_t(t)];
    const int32_t s0 = int32_t(o_s[size_t(t)]);
    std::copy(x.segs.begin(), x.segs.end(), ga.segs.begin() + o_s[size_t(t)]);
    for (size_t k = 0; k < x.tiles.size(); ++k) {
      GTile gt = x.tiles[k];
      gt.seg_begin += s0;
      gt.seg_end += s0;
      ga.tiles[o_x[size_t(t)] + k] = gt;
    }
  };
  std::vector<std::thread> mt;
  for (int t = 1; t < nt; ++t) mt.emplace_back(merge, t);
  merge(0);
  for (auto& x : mt) x.join();
}

// ----------------------------------------------------------------------------- context
struct hx_ctx {
  // page-locked staging of the product's small device-to-host reads (ranks, flags, norms):
  // a copy into pageable memory goes through the driver's shared staging path and was seen
  // waiting ~60 ms behind other contexts' transfers
  void* stage = nullptr;
  size_t stage_bytes = 0;
  void d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (!bytes) return;
    if (bytes > stage_bytes) {
      if (stage) hx::pinned_free(stage, stage_bytes);
      stage_bytes = std::max(bytes, size_t(1) << 20);
      stage = hx::pinned_alloc(stage_bytes);
    }
    CK(cudaMemcpyAsync(stage, src, bytes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::memcpy(dst, stage, bytes);
  }
  int device = 0;
  cudaStream_t s = nullptr;
  cudaStream_t s2 = nullptr;  // copy stream (materialization work lists)
  // high-priority stream for the latency-bound recompression: when two contexts run
  // consecutive chunks, its small launches get SMs ahead of the other chunk's formation
  cudaStream_t s_hi = nullptr;
  cudaStream_t s3 = nullptr;  // second formation stream (odd batches)
  DArr<double> own[NUM_BUFS];
  double* attached[2] = {nullptr, nullptr};
  int64_t opnd_elems[2] = {0, 0};
  bool alias = false;
  DArr<Term> terms[3];
  DArr<Tile> tiles[3];
  DArr<Group> groups[3];
  DArr<double> sumsq, fro2;
  DArr<int> seg_b, seg_e;
  DArr<ColRec> gcols;
  DArr<TransRec> trans_recs;
  bool eye_ready = false;
  DArr<Term> rterms;
  DArr<Tile> rtiles;
  DArr<Group> rgroups;
  DArr<QrJob> qr_jobs;
  DArr<TsMul> ts_jobs;     // TSQR down-sweep slabs
  DArr<double> tsqr_ws;    // TSQR stacked R factors
  DArr<JacJob> jac_jobs;
  DArr<SelJob> sel_jobs;
  DArr<SmallJob> small_jobs;
  DArr<int> rank_d, retry_d;
  DArr<double> rsum, resid;  // explicit-tail sums of squares (per tile, per block)
  DArr<double> esum, est;    // implicit route: probe residual sums (per tile, per block)
  DArr<int> tb, te, eb, ee;
  DArr<Term> xterms;         // one upload of all grouped-GEMM batches of a sketch round
  DArr<Tile> xtiles;
  DArr<Group> xgroups;
  DArr<GTile> gtiles;        // row-gathered GEMM tiles / segments of a sketch round
  DArr<GSeg> gsegs;
  DArr<IterJob> iter_jobs;   // matrix-free compressors (aca / bilanczos / randomized)
  DArr<IterTerm> iter_terms;
  DArr<IterOut> iter_outs;
  DArr<UrJob> ur_jobs;
  std::vector<DArr<double>> work;  // one workspace per sketch round
  // traditional mode (traditional_exec.cuh): wave workspace, ping-pong running sums, kept
  // values of finished folds, wave work lists
  DArr<double> trad_ws, trad_tmp[2], trad_nv;
  std::vector<DArr<double>> trad_keep;
  DArr<TSeg> trad_segs;
  DArr<TNormJob> trad_norm_jobs;
  DArr<const double*> trad_sigp;
  void trad_release(bool all) {
    for (auto& k : trad_keep) k.release();
    trad_keep.clear();
    if (!all) return;
    trad_ws.release();
    trad_tmp[0].release();
    trad_tmp[1].release();
    trad_nv.release();
    trad_segs.release();
    trad_norm_jobs.release();
    trad_sigp.release();
  }
  std::vector<double*> pools;      // operand pools built by hx_assemble (owned)
  // sketch-width hints: the largest rank seen per log2(min(m, n)) class by earlier chunks
  // of the same product (hx_ctx_reset_hints between products), for the same policy
  int rank_hint[32];
  int8_t class_retry[32];  // a block of the class needed a wider sketch (retry round)
  // matrix-free compressors: the most columns a block of the class produced (before the
  // final truncation) in earlier chunks; the next chunks size their column budget from it
  // instead of rerunning capped blocks with four times the budget
  int iter_hint[32];
  double hint_key[4] = {-1, -1, -1, -1};
  int64_t omega_rows = 0;
  int omega_cols = 0;
  uint64_t omega_seed = ~0ULL;
  // results
  std::vector<int32_t> res_rank;
  std::vector<int8_t> res_deg;
  std::vector<int64_t> res_off;
  int64_t out_far = 0, near_begin = 0, near_elems = 0;
  int64_t launches = 0;
  cudaEvent_t ev[8];
  cudaEvent_t up_ev = nullptr;  // end of the last host-to-device operand copy on s

  double* buf(int i) {
    if (i == BUF_A) return attached[0] ? attached[0] : own[BUF_A].p;
    if (i == BUF_B) {
      if (alias) return buf(BUF_A);
      return attached[1] ? attached[1] : own[BUF_B].p;
    }
    return own[i].p;
  }
  BufPtrs ptrs() {
    BufPtrs b;
    for (int i = 0; i < NUM_BUFS; ++i) b.p[i] = buf(i);
    return b;
  }
};

namespace {

void launch_gemm(hx_ctx* c, int tile, const Tile* tiles, const Group* groups, const Term* terms,
                 int n_tiles, const BufPtrs& bp, double* sumsq,
                 const ColRec* gcols = nullptr, bool short_k = false,
                 cudaStream_t stream = nullptr) {
  if (n_tiles <= 0) return;
  cudaStream_t st = stream ? stream : c->s;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(grouped_gemm_kernel<Gemm64>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, Gemm64::SMEM));
    CK(cudaFuncSetAttribute(grouped_gemm_kernel<Gemm32>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, Gemm32::SMEM));
    CK(cudaFuncSetAttribute(grouped_gemm_kernel<Gemm64s>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, Gemm64s::SMEM));
    attr = true;
  }
  static const bool use_short = !std::getenv("HX_NO_SHORTK");
  // warp-specialized persistent kernel (gemm_ws.cuh) unless HX_GEMM_WS=0
  static const bool use_ws = !(std::getenv("HX_GEMM_WS") && std::getenv("HX_GEMM_WS")[0] == '0');
  if (tile == 64 && use_ws) {
    // grids: one CTA per resident slot.  HX_WS_RESERVE: SMs left free of the persistent
    // GEMM CTAs (for the latency-bound recompression of a concurrent chunk on another context)
    static int grid[2][2] = {{0, 0}, {0, 0}};  // [short K][column records]
    if (!grid[0][0]) {
      static const int reserve = std::getenv("HX_WS_RESERVE") ? std::atoi(std::getenv("HX_WS_RESERVE")) : 0;
      auto grid_of = [](auto kern, int threads, int smem) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int dev = 0, sms = 0, b = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, smem));
        return std::max(1, b) * std::max(1, sms - reserve);
      };
      grid[0][0] = grid_of(grouped_gemm_ws_kernel<Ws64, false>, Ws64::THREADS, Ws64::SMEM);
      grid[0][1] = grid_of(grouped_gemm_ws_kernel<Ws64, true>, Ws64::THREADS, Ws64::SMEM);
      grid[1][0] = grid_of(grouped_gemm_ws_kernel<Ws64s, false>, Ws64s::THREADS, Ws64s::SMEM);
      grid[1][1] = grid_of(grouped_gemm_ws_kernel<Ws64s, true>, Ws64s::THREADS, Ws64s::SMEM);
    }
    const bool sk = short_k && use_short, gc = gcols != nullptr;
    const int g = std::min(n_tiles, grid[sk][gc]);
    if (sk && gc)
      grouped_gemm_ws_kernel<Ws64s, true><<<g, Ws64s::THREADS, Ws64s::SMEM, st>>>(
          tiles, groups, terms, bp, sumsq, n_tiles, gcols);
    else if (sk)
      grouped_gemm_ws_kernel<Ws64s, false><<<g, Ws64s::THREADS, Ws64s::SMEM, st>>>(
          tiles, groups, terms, bp, sumsq, n_tiles, gcols);
    else if (gc)
      grouped_gemm_ws_kernel<Ws64, true><<<g, Ws64::THREADS, Ws64::SMEM, st>>>(
          tiles, groups, terms, bp, sumsq, n_tiles, gcols);
    else
      grouped_gemm_ws_kernel<Ws64, false><<<g, Ws64::THREADS, Ws64::SMEM, st>>>(
          tiles, groups, terms, bp, sumsq, n_tiles, gcols);
    CK(cudaGetLastError());
    c->launches++;
    return;
  }
  if (tile == 64 && short_k && use_short)
    grouped_gemm_kernel<Gemm64s><<<n_tiles, Gemm64s::THREADS, Gemm64s::SMEM, st>>>(
        tiles, groups, terms, bp, sumsq, n_tiles, gcols);
  else if (tile == 32)
    grouped_gemm_kernel<Gemm32><<<n_tiles, Gemm32::THREADS, Gemm32::SMEM, st>>>(
        tiles, groups, terms, bp, sumsq, n_tiles, gcols);
  else
    grouped_gemm_kernel<Gemm64><<<n_tiles, Gemm64::THREADS, Gemm64::SMEM, st>>>(
        tiles, groups, terms, bp, sumsq, n_tiles, gcols);
  CK(cudaGetLastError());
  c->launches++;
}

// Tiles for out (R x C, ld R) = P * Q with a single term.
void single_term_tiles(std::vector<Term>& terms, std::vector<Tile>& tiles,
                       std::vector<Group>& groups, const Term& t, uint8_t out_buf,
                       int64_t out_off, int R, int C) {
  const int32_t g = int32_t(groups.size());
  groups.push_back(Group{int32_t(terms.size()), int32_t(terms.size()) + 1});
  terms.push_back(t);
  for (int j = 0; j < C; j += 64)
    for (int i = 0; i < R; i += 64) {
      Tile tl;
      std::memset(&tl, 0, sizeof(tl));
      tl.out_off = out_off + i + int64_t(j) * R;
      tl.out_ld = R;
      tl.row0 = i;
      tl.col0 = j;
      tl.rows = int16_t(std::min(64, R - i));
      tl.cols = int16_t(std::min(64, C - j));
      tl.g_begin = g;
      tl.g_end = g + 1;
      tl.aux = -1;
      tl.out_buf = out_buf;
      tl.mode = MODE_STORE;
      tiles.push_back(tl);
    }
}

Term mk(uint8_t abuf, int64_t aoff, int32_t ald, uint8_t akc, uint8_t bbuf, int64_t boff,
        int32_t bld, uint8_t bkc, int32_t k, int32_t rows, int32_t cols) {
  Term t;
  t.a_off = aoff;
  t.b_off = boff;
  t.a_ld = ald;
  t.b_ld = bld;
  t.k = k;
  t.r_lo = 0;
  t.c_lo = 0;
  t.rows = rows;
  t.cols = cols;
  t.a_buf = abuf;
  t.b_buf = bbuf;
  t.a_kc = akc;
  t.b_kc = bkc;
  return t;
}

void run_gemm_batch(hx_ctx* c, std::vector<Term>& terms, std::vector<Tile>& tiles,
                    std::vector<Group>& groups) {
  if (tiles.empty()) return;
  c->rterms.upload(terms, c->s);
  c->rtiles.upload(tiles, c->s);
  c->rgroups.upload(groups, c->s);
  launch_gemm(c, 64, c->rtiles.p, c->rgroups.p, c->rterms.p, int(tiles.size()), c->ptrs(),
              nullptr);
}

// QR jobs: small panels (p <= 256, q <= 32) one warp each, others one CTA each (panel in
// shared memory when it fits, else in place in HBM/L2).
// Row-parallel Householder QR (qr_rows.cuh): panels up to QR_WARP_ROWS rows one warp each
// (bucketed by height so that each launch sizes its smem slices tightly), taller ones one
// CTA each, in shared memory when the panel fits.
constexpr int QR_WARP_ROWS = 128;
// TSQR row blocks of b..2b-1 rows: b = 128 for q <= 32 (blocks go to the register QR
// kernel), else the tallest b <= 256 whose 2b-row block still fits the shared-memory QR
// (HX_TSQR_BLOCK overrides)
int ts_block(int q) {
  static const int env = std::getenv("HX_TSQR_BLOCK") ? std::atoi(std::getenv("HX_TSQR_BLOCK"))
                                                      : 0;
  if (env > 0) return env;
  if (q <= 32) return 128;
  const int fit = int(size_t(SMEM_CAP) / (8 * size_t(q) + 8)) / 2;
  return std::max(64, std::min(256, fit & ~7));
}

// Shared memory bounds occupancy here, so jobs are bucketed by their smem need (powers of
// two) and every launch sizes its slices for its own bucket.
// Bucket, sort and launch one set of independent QR jobs (already uploaded at dev).
void launch_qr_set(hx_ctx* c, const QrJob* dev, const std::vector<QrJob>& all,
                   const std::vector<int>& keys, size_t a0, size_t a1);

int qr_bucket(const QrJob& j);

void run_qr(hx_ctx* c, const std::vector<QrJob>& jobs) {
  if (jobs.empty()) return;
  // TSQR decomposition of the tall panels (qr_rows.cuh): up-sweep levels of QR jobs and
  // down-sweep slab products; offsets into one workspace, sized before any pointer is taken
  // panels above 512 rows (config 2: the 1024-blocks' sketches, which overflow shared
  // memory; recompression 89 -> 80 ms) and the very tall panels of the largest blocks
  static const int ts_min = std::getenv("HX_TSQR_MIN") ? std::atoi(std::getenv("HX_TSQR_MIN"))
                                                       : 512;
  static const bool no_tsqr = std::getenv("HX_NO_TSQR") != nullptr;
  auto tall = [](const QrJob& j) {
    return !no_tsqr && j.q <= TS_QMAX && j.p > std::max(ts_min, 2 * ts_block(j.q));
  };
  int64_t ws = 0;
  for (const QrJob& j : jobs) {
    if (!tall(j)) continue;
    int64_t p = j.p;
    const int tb = ts_block(j.q);
    while (p > 2 * tb) {
      const int64_t nb = p / tb;
      ws += nb * j.q * j.q;
      p = nb * j.q;
    }
  }
  if (ws) c->tsqr_ws.ensure(size_t(ws));
  std::vector<std::vector<QrJob>> lev(1);
  std::vector<std::vector<TsMul>> down;
  int64_t pos = 0;
  for (const QrJob& j : jobs) {
    if (!tall(j)) {
      lev[0].push_back(j);
      continue;
    }
    double* X = j.X;
    int ld = j.lx();
    int p = j.p;
    const int q = j.q;
    for (size_t L = 0;; ++L) {
      if (lev.size() <= L) lev.resize(L + 1);
      if (p <= 2 * ts_block(q)) {
        QrJob t{X, j.R, p, q};
        t.ldx = ld;
        t.ldr = j.lr();
        lev[L].push_back(t);
        break;
      }
      if (down.size() <= L) down.resize(L + 1);
      const int nb = p / ts_block(q);
      const int ls = nb * q;  // rows (and ld) of the stacked R factors
      double* S = c->tsqr_ws.p + pos;
      pos += int64_t(ls) * q;
      const int base = p / nb, extra = p % nb;
      int r0 = 0;
      for (int i = 0; i < nb; ++i) {
        const int rows = base + (i < extra ? 1 : 0);
        QrJob t{X + r0, S + int64_t(i) * q, rows, q};
        t.ldx = ld;
        t.ldr = ls;
        lev[L].push_back(t);
        for (int s0 = 0; s0 < rows; s0 += TS_SLAB)
          down[L].push_back(TsMul{X + r0 + s0, S + int64_t(i) * q, ld, ls,
                                  std::min(TS_SLAB, rows - s0), q});
        r0 += rows;
      }
      X = S;
      ld = ls;
      p = ls;
    }
  }
  std::vector<QrJob> all;
  std::vector<int> keys;
  std::vector<size_t> lb;
  for (auto& L : lev) {
    lb.push_back(all.size());
    std::vector<std::pair<int, int>> keyed(L.size());
    for (size_t i = 0; i < L.size(); ++i) keyed[i] = {qr_bucket(L[i]), int(i)};
    std::sort(keyed.begin(), keyed.end());
    for (auto& kv : keyed) {
      all.push_back(L[size_t(kv.second)]);
      keys.push_back(kv.first);
    }
  }
  lb.push_back(all.size());
  c->qr_jobs.upload(all, c->s);
  std::vector<TsMul> dm;
  std::vector<size_t> db;
  for (auto& D : down) {
    db.push_back(dm.size());
    dm.insert(dm.end(), D.begin(), D.end());
  }
  db.push_back(dm.size());
  if (!dm.empty()) c->ts_jobs.upload(dm, c->s);
  for (size_t L = 0; L + 1 < lb.size(); ++L) launch_qr_set(c, c->qr_jobs.p, all, keys, lb[L], lb[L + 1]);
  static bool tattr = false;
  if (!dm.empty() && !tattr) {
    CK(cudaFuncSetAttribute(tsqr_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(2 * TS_SLAB * TS_QMAX * sizeof(double))));
    tattr = true;
  }
  for (size_t L = down.size(); L-- > 0;) {
    const size_t n = db[L + 1] - db[L];
    if (!n) continue;
    tsqr_apply_kernel<<<int(n), 256, 2 * TS_SLAB * TS_QMAX * sizeof(double), c->s>>>(
        c->ts_jobs.p + db[L]);
    CK(cudaGetLastError());
    c->launches++;
  }
}

// register-resident kernel: q <= 32, p <= 256; key 192 + 4 (QM == 32) + log2(NW) with
// two rows per thread for QM = 16 and one for QM = 32
bool qr_reg_job(const QrJob& j) { return j.q <= 32 && j.q <= j.p && j.p <= 256; }
size_t qr_slice(const QrJob& j) { return size_t(j.p) * j.q + j.q + 32; }  // doubles
bool qr_warp_job(const QrJob& j) {
  return j.p <= QR_WARP_ROWS && qr_slice(j) * sizeof(double) <= size_t(SMEM_CAP);
}

// bucket key: kind (0 warp, 1 CTA smem, 2 CTA global, 3 register) and log2 of the smem bytes
int qr_bucket(const QrJob& j) {
  auto lg_nw = [](int rows_per_warp, int p) {
    int l = 0;
    while ((rows_per_warp << l) < p) ++l;
    return l;
  };
  if (qr_reg_job(j)) return j.q > 16 ? 196 + lg_nw(32, j.p) : 192 + lg_nw(64, j.p);
  const size_t need = qr_warp_job(j) ? qr_slice(j) * sizeof(double)
                                     : size_t(j.p) * j.q * sizeof(double);
  const int kind = qr_warp_job(j) ? 0 : (need <= size_t(SMEM_CAP) ? 1 : 2);
  int lg = 0;
  while ((size_t(1) << lg) < need && lg < 40) ++lg;
  return kind == 2 ? 2 * 64 : kind * 64 + lg;
}

void launch_qr_set(hx_ctx* c, const QrJob* dev, const std::vector<QrJob>& all,
                   const std::vector<int>& keys, size_t a0, size_t a1) {
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(qr_rows_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(SMEM_CAP)));
    CK(cudaFuncSetAttribute(qr_rows_cta_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(SMEM_CAP)));
    CK(cudaFuncSetAttribute(qr_rows_cta_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(SMEM_CAP)));
    attr = true;
  }
  for (size_t a = a0; a < a1;) {
    size_t e = a;
    size_t need = 0;
    while (e < a1 && keys[e] == keys[a]) {
      need = std::max(need, qr_warp_job(all[e]) ? qr_slice(all[e])
                                                : size_t(all[e].p) * all[e].q);
      ++e;
    }
    const int n = int(e - a);
    const int kind = keys[a] / 64;
    const QrJob* jp = dev + a;
    if (kind == 3) {
      switch (keys[a] - 192) {
        case 0: qr_reg_kernel<1, 16, 2><<<n, 32, 0, c->s>>>(jp); break;
        case 1: qr_reg_kernel<2, 16, 2><<<n, 64, 0, c->s>>>(jp); break;
        case 2: qr_reg_kernel<4, 16, 2><<<n, 128, 0, c->s>>>(jp); break;
        case 4: qr_reg_kernel<1, 32, 1><<<n, 32, 0, c->s>>>(jp); break;
        case 5: qr_reg_kernel<2, 32, 1><<<n, 64, 0, c->s>>>(jp); break;
        case 6: qr_reg_kernel<4, 32, 1><<<n, 128, 0, c->s>>>(jp); break;
        default: qr_reg_kernel<8, 32, 1><<<n, 256, 0, c->s>>>(jp); break;
      }
    } else if (kind == 0) {
      const size_t per = need * sizeof(double);
      const int wpc = int(std::max<size_t>(1, std::min<size_t>(4, size_t(SMEM_CAP) / per)));
      qr_rows_warp_kernel<<<(n + wpc - 1) / wpc, 32 * wpc, per * size_t(wpc), c->s>>>(
          jp, n, int(need));
    } else if (kind == 1) {
      if (all[a].p > 256)
        qr_rows_cta_kernel<512><<<n, 512, need * sizeof(double), c->s>>>(jp, 1);
      else
        qr_rows_cta_kernel<256><<<n, 256, need * sizeof(double), c->s>>>(jp, 1);
    } else {
      qr_rows_cta_kernel<512><<<n, 512, 0, c->s>>>(jp, 0);
    }
    CK(cudaGetLastError());
    c->launches++;
    a = e;
  }
}

// Jacobi jobs: q <= 16 / q <= 32 one warp each (columns in registers), larger one CTA.
void run_jacobi(hx_ctx* c, const std::vector<JacJob>& jobs) {
  if (jobs.empty()) return;
  std::vector<JacJob> all;
  all.reserve(jobs.size());
  for (const JacJob& j : jobs)
    if (j.q <= 16) all.push_back(j);
  const size_t n16 = all.size();
  for (const JacJob& j : jobs)
    if (j.q > 16 && j.q <= 32) all.push_back(j);
  const size_t n32 = all.size() - n16;
  int qmax = 0;
  for (const JacJob& j : jobs)
    if (j.q > 32) {
      all.push_back(j);
      qmax = std::max(qmax, j.q);
    }
  const size_t nb = all.size() - n16 - n32;
  c->jac_jobs.upload(all, c->s);
  if (n16) {
    warp_jacobi_kernel<16><<<int((n16 + 3) / 4), 128, 0, c->s>>>(c->jac_jobs.p, int(n16));
    CK(cudaGetLastError());
    c->launches++;
  }
  if (n32) {
    warp_jacobi_kernel<32><<<int((n32 + 3) / 4), 128, 0, c->s>>>(c->jac_jobs.p + n16, int(n32));
    CK(cudaGetLastError());
    c->launches++;
  }
  if (nb) {
    const int qs = std::min(qmax, JAC_SMEM_QMAX);  // wider factors run in place in HBM
    const size_t smem = size_t(2) * qs * qs * sizeof(double);
    CK(cudaFuncSetAttribute(jacobi_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            int(std::max<size_t>(smem, 1))));
    // one warp per column pair of a round (widest job), 8..32 warps
    static const int wide = std::getenv("HX_JAC_WIDE") ? std::atoi(std::getenv("HX_JAC_WIDE")) : 1;
    const int nt = wide ? 32 * std::max(8, std::min(32, (qmax + 1) / 2)) : LA_THREADS;
    jacobi_svd_kernel<<<int(nb), nt, smem, c->s>>>(c->jac_jobs.p + n16 + n32);
    CK(cudaGetLastError());
    c->launches++;
  }
}

int ilog2(int x) {
  int l = 0;
  while ((1 << (l + 1)) <= x && l < 31) ++l;
  return l;
}

int default_sketch(int mu) {
  // first sketch width by block size (64, 128, 256, 512, larger); HX_SKETCH_TABLE overrides
  // (config 2: 16,24,32,40,48 -> 16,24,32,32,40 cuts recompression 79 -> 76 ms without
  // extra retry rounds; classes that do retry widen through the rank hints)
  static const std::vector<int> tab = [] {
    std::vector<int> t{16, 24, 32, 32, 40};
    if (const char* e = std::getenv("HX_SKETCH_TABLE")) {
      std::vector<int> u;
      for (const char* p = e; *p;) {
        u.push_back(std::atoi(p));
        while (*p && *p != ',') ++p;
        if (*p) ++p;
      }
      if (u.size() == t.size()) t = u;
    }
    return t;
  }();
  if (mu <= 64) return tab[0];
  if (mu <= 128) return tab[1];
  if (mu <= 256) return tab[2];
  if (mu <= 512) return tab[3];
  return tab[4];
}

// First column budget of the matrix-free compressors by block size (a block that needs
// more is rerun with four times as many; ACA and Lanczos are deterministic per block).
int iter_kcap0(int mu) {
  if (mu <= 64) return 24;
  if (mu <= 128) return 32;
  if (mu <= 256) return 48;
  if (mu <= 1024) return 64;
  return 96;
}

// Far blocks compressed by the reference's matrix-free schemes (the aca / bilanczos /
// randomized tags; compressors.py:162-428) on their implicit sums, then the exact SVD
// recompressions those schemes end with.  Fills f.Y / f.Bt / f.R / f.W / f.V / f.sig / f.l
// (SVD-finished blocks, like the sketch route) or sets f.direct (factors output as
// produced), f.rank and f.degraded; returns the reference's matvec count.
int64_t recompress_iterative(hx_ctx* c, hx_plan* P, const hx_product_cfg* cfg,
                             std::vector<FarBlock>& fb, int jac_trans, int& rounds) {
  const int nf = int(fb.size());
  int64_t matvecs = 0;
  if (!nf) return 0;
  const int tag = cfg->tag;  // 0 aca, 1 bilanczos, 2 randomized
  IterParams prm;
  prm.tag = tag == 0 ? ITER_ACA : (tag == 1 ? ITER_GKL : ITER_RAND);
  prm.policy = cfg->policy;
  prm.eps = cfg->eps;
  prm.k_max = cfg->k_max;
  prm.q = cfg->q;
  prm.seed = cfg->seed;
  const BufPtrs bp0 = c->ptrs();
  // terms of the implicit blocks, clipped to the block (leaf-local coordinates)
  std::vector<IterTerm> terms;
  std::vector<int> tbeg(nf, 0), tend(nf, 0), ksum(nf, 0);
  for (int i = 0; i < nf; ++i) {
    FarBlock& f = fb[size_t(i)];
    tbeg[size_t(i)] = int(terms.size());
    if (f.implicit) {
      const OutLeaf& L = P->leaves[size_t(f.leaf)];
      int koff = 0;
      for (const ImplTerm& x : f.it) {
        const Term& t = x.t;
        if (t.b_kc > 1 || t.a_kc > 1) throw hx::Unsupported("gathered term on the implicit route");
        for (uint8_t b : {t.a_buf, t.b_buf})
          if (b == BUF_CORE || b == BUF_WORK || b == BUF_OUT)
            throw hx::Unsupported("implicit term on a transient buffer");
        IterTerm e;
        const int64_t ri = L.row0 + x.ri - t.r_lo;  // term-local first row / column
        const int64_t cj = L.col0 + x.ci - t.c_lo;
        e.ps = t.a_kc ? t.a_ld : 1;
        e.pk = t.a_kc ? 1 : t.a_ld;
        e.qs = t.b_kc ? t.b_ld : 1;
        e.qk = t.b_kc ? 1 : t.b_ld;
        e.P = bp0.p[t.a_buf] + t.a_off + ri * e.ps;
        e.Q = bp0.p[t.b_buf] + t.b_off + cj * e.qs;
        e.k = x.k;
        e.ri = x.ri;
        e.rn = x.rn;
        e.ci = x.ci;
        e.cn = x.cn;
        e.koff = koff;
        koff += x.k;
        terms.push_back(e);
      }
      // the block-sparse T_sub: every dense block as a term T_b I (identity from BUF_EYE)
      for (int32_t q = L.tsub_begin; q < L.tsub_end; ++q) {
        const TSubBlock& tb = P->tsub[size_t(q)];
        if (tb.w > EYE_LD) throw hx::Unsupported("T_sub block wider than the identity buffer");
        IterTerm e;
        e.P = bp0.p[BUF_TILE] + tb.off;
        e.ps = 1;
        e.pk = tb.h;
        e.Q = bp0.p[BUF_EYE];
        e.qs = EYE_LD;
        e.qk = 1;
        e.k = tb.w;
        e.ri = int32_t(tb.r0 - L.row0);
        e.rn = tb.h;
        e.ci = int32_t(tb.c0 - L.col0);
        e.cn = tb.w;
        e.koff = koff;
        koff += tb.w;
        terms.push_back(e);
      }
      ksum[size_t(i)] = koff;
    }
    tend[size_t(i)] = int(terms.size());
  }
  if (!terms.empty()) c->iter_terms.upload(terms, c->s);
  std::vector<int> kcap(nf);
  for (int i = 0; i < nf; ++i) {
    const FarBlock& f = fb[size_t(i)];
    int k0 = iter_kcap0(f.mu);
    const int h = c->iter_hint[ilog2(f.mu)];
    if (h >= 0) k0 = std::max(k0, (h + 8 + 7) & ~7);
    kcap[size_t(i)] = cfg->policy == 1 ? std::min(f.mu, std::max(cfg->k_max, 1))
                                       : std::min(f.mu, k0);
  }
  auto a16 = [](int64_t x) { return (x + 15) & ~int64_t(15); };
  std::vector<IterOut> outs(static_cast<size_t>(nf));
  std::vector<int> active(static_cast<size_t>(nf));
  for (int i = 0; i < nf; ++i) active[size_t(i)] = i;
  std::vector<IterJob> jobs(static_cast<size_t>(nf));
  // job workspace offsets (doubles) in c->work[0]; re-laid out per round of reruns
  while (!active.empty()) {
    if (rounds >= 6) throw std::runtime_error("matrix-free compression did not converge");
    int64_t wsz = 0;
    std::vector<int64_t> off(active.size());
    for (size_t a = 0; a < active.size(); ++a) {
      const int i = active[a];
      const FarBlock& f = fb[size_t(i)];
      const int64_t kc = kcap[size_t(i)];
      off[a] = wsz;
      wsz += a16(f.m * kc) + a16(f.n * kc) + (tag == 1 ? a16(f.n * kc) : 0) + a16(2 * f.m) +
             a16(3 * int64_t(f.n)) + a16(((ksum[size_t(i)] + 7) & ~7) + 2 * kc + 8) +
             a16((f.m + f.n + 7) / 8);
    }
    const int slot = rounds;  // finished jobs of earlier rounds keep their slots
    if (int(c->work.size()) <= slot) c->work.resize(slot + 1);
    c->work[slot].ensure(size_t(std::max<int64_t>(wsz, 16)));
    double* wb = c->work[slot].p;
    // large / implicit blocks: a CTA of 8 warps each; the others a warp each
    std::vector<int> big, small;
    for (size_t a = 0; a < active.size(); ++a) {
      const int i = active[a];
      FarBlock& f = fb[size_t(i)];
      const int64_t kc = kcap[size_t(i)];
      double* p = wb + off[a];
      IterJob jb;
      jb.T = f.implicit ? nullptr : c->buf(BUF_TILE) + f.t_off;
      jb.ldT = f.m;
      jb.m = f.m;
      jb.n = f.n;
      jb.t_begin = tbeg[size_t(i)];
      jb.t_end = tend[size_t(i)];
      jb.kcap = int32_t(kc);
      jb.node = P->leaves[size_t(f.leaf)].id;
      jb.L = p;
      p += a16(f.m * kc);
      jb.U = p;
      p += a16(f.n * kc);
      jb.Wb = nullptr;
      if (tag == 1) {
        jb.Wb = p;
        p += a16(f.n * kc);
      }
      jb.vm = p;
      p += a16(2 * f.m);
      jb.vn = p;
      p += a16(3 * int64_t(f.n));
      jb.tz = p;
      p += a16(((ksum[size_t(i)] + 7) & ~7) + 2 * kc + 8);
      jb.used = reinterpret_cast<uint8_t*>(p);
      jobs[size_t(i)] = jb;
      (f.implicit || std::max(f.m, f.n) > 256 ? big : small).push_back(i);
    }
    auto by_size = [&](int x, int y) {
      const int64_t ax = int64_t(fb[size_t(x)].m) * fb[size_t(x)].n;
      const int64_t ay = int64_t(fb[size_t(y)].m) * fb[size_t(y)].n;
      return ax != ay ? ax > ay : x < y;
    };
    std::sort(big.begin(), big.end(), by_size);
    std::sort(small.begin(), small.end(), by_size);
    std::vector<IterJob> order;
    for (int i : big) order.push_back(jobs[size_t(i)]);
    for (int i : small) order.push_back(jobs[size_t(i)]);
    c->iter_jobs.upload(order, c->s);
    c->iter_outs.ensure(order.size());
    if (!big.empty()) {
      iter_kernel<8><<<int(big.size()), 256, 0, c->s>>>(c->iter_jobs.p, c->iter_terms.p,
                                                         c->iter_outs.p, int(big.size()), prm);
      CK(cudaGetLastError());
      c->launches++;
    }
    if (!small.empty()) {
      iter_kernel<1><<<int((small.size() + 3) / 4), 128, 0, c->s>>>(
          c->iter_jobs.p + big.size(), c->iter_terms.p, c->iter_outs.p + big.size(),
          int(small.size()), prm);
      CK(cudaGetLastError());
      c->launches++;
    }
    std::vector<IterOut> got(order.size());
    c->d2h(got.data(), c->iter_outs.p, got.size() * sizeof(IterOut), c->s);
    std::vector<int> next;
    size_t a = 0;
    for (int i : big) outs[size_t(i)] = got[a++];
    for (int i : small) outs[size_t(i)] = got[a++];
    for (int i : active) {
      const FarBlock& f = fb[size_t(i)];
      if (outs[size_t(i)].capped && kcap[size_t(i)] < f.mu) {
        kcap[size_t(i)] = std::min(f.mu, 4 * kcap[size_t(i)]);
        next.push_back(i);
      } else if (outs[size_t(i)].capped) {
        throw std::runtime_error("matrix-free compression: column budget exhausted");
      }
    }
    ++rounds;
    if (next.empty()) break;
    active.swap(next);
  }
  for (int i = 0; i < nf; ++i) {
    matvecs += outs[size_t(i)].matvecs;
    int& h = c->iter_hint[ilog2(fb[size_t(i)].mu)];
    h = std::max(h, outs[size_t(i)].k);
  }
  // ---- exact recompressions: ACA's truncate(eps / 2) (compressors.py:245-246,
  // lowrank.py:93-113) and the Lanczos core SVD (:359-365); the sketch route's kernels
  int64_t psz = 0;
  std::vector<int> svd;
  for (int i = 0; i < nf; ++i) {
    FarBlock& f = fb[size_t(i)];
    const IterOut& o = outs[size_t(i)];
    f.degraded = o.degraded;
    f.done = 1;
    f.rank = o.k;
    f.l = o.k;
    f.dense = 0;
    f.Y = jobs[size_t(i)].L;
    f.Bt = jobs[size_t(i)].U;
    const bool trunc = o.k > 0 && ((tag == 0 && cfg->policy == 0 && o.k > 1) || tag == 1);
    if (!trunc) {
      f.direct = 1;
      continue;
    }
    if (o.k > JAC_QMAX) throw hx::Unsupported("compressed block rank above " +
                                              std::to_string(JAC_QMAX));
    svd.push_back(i);
    const int64_t k = o.k;
    psz += 4 * a16(k * k) + a16(k) + (tag == 0 ? a16(int64_t(f.n) * k) : 0);
  }
  if (svd.empty()) return matvecs;
  const int post = rounds;
  if (int(c->work.size()) <= post) c->work.resize(post + 1);
  c->work[post].ensure(size_t(std::max<int64_t>(psz, 16)));
  double* wb = c->work[post].p;
  int64_t pos = 0;
  auto take = [&](int64_t ne) {
    double* p = wb + pos;
    pos += a16(ne);
    return p;
  };
  std::vector<QrJob> q1, q2;
  std::vector<UrJob> ur;
  for (int i : svd) {
    FarBlock& f = fb[size_t(i)];
    const int k = f.l;
    f.R = take(int64_t(k) * k);
    f.W = take(int64_t(k) * k);
    f.V = take(int64_t(k) * k);
    f.sig = take(k);
    if (tag == 0) {
      // L = Q_L R_L (in place); Bt = U R_L^T = (L U^T)^T Q_L, then Bt = Q2 R as on the
      // sketch route
      double* rl = take(int64_t(k) * k);
      q1.push_back(QrJob{f.Y, rl, f.m, k});
      double* bt = take(int64_t(f.n) * k);
      ur.push_back(UrJob{f.Bt, rl, bt, f.n, k});
      f.Bt = bt;
    }
  }
  if (tag == 0) {
    run_qr(c, q1);
    c->ur_jobs.upload(ur, c->s);
    int nmax = 1;
    for (const UrJob& u : ur) nmax = std::max(nmax, u.n);
    dim3 grid(unsigned(ur.size()), unsigned(std::min(64, (nmax + 127) / 128)));
    ur_product_kernel<<<grid, 128, 0, c->s>>>(c->ur_jobs.p);
    CK(cudaGetLastError());
    c->launches++;
  }
  for (int i : svd) {
    FarBlock& f = fb[size_t(i)];
    q2.push_back(QrJob{const_cast<double*>(f.Bt), f.R, f.n, f.l});
  }
  run_qr(c, q2);
  std::vector<JacJob> jj;
  for (int i : svd) {
    FarBlock& f = fb[size_t(i)];
    jj.push_back(JacJob{f.R, f.sig, f.W, f.V, f.l, jac_trans});
  }
  run_jacobi(c, jj);
  std::vector<SelJob> sj;
  for (int i : svd) {
    FarBlock& f = fb[size_t(i)];
    sj.push_back(SelJob{f.sig, nullptr, f.l, f.mu, 1, 0});
  }
  const int na = int(sj.size());
  c->sel_jobs.upload(sj, c->s);
  c->rank_d.ensure(size_t(na));
  c->retry_d.ensure(size_t(na));
  // ACA trims at eps / 2; Lanczos selects at eps (FixedRank keeps min(k, k_max))
  const double eps_sel = tag == 0 ? 0.5 * cfg->eps : cfg->eps;
  select_rank_kernel<<<(na + 127) / 128, 128, 0, c->s>>>(c->sel_jobs.p, na, cfg->policy, eps_sel,
                                                         cfg->k_max, 0, c->rank_d.p,
                                                         c->retry_d.p, 0);
  CK(cudaGetLastError());
  c->launches++;
  std::vector<int> rk(static_cast<size_t>(na));
  c->d2h(rk.data(), c->rank_d.p, size_t(na) * sizeof(int), c->s);
  for (int a = 0; a < na; ++a) fb[size_t(svd[size_t(a)])].rank = rk[size_t(a)];
  return matvecs;
}

// Output factors of the far blocks: left (m x r) = U S and right (n x r) = V written at
// out + off[i] (left then right, column-major), from the recompression's small factors.
void launch_far_outputs(hx_ctx* c, const std::vector<FarBlock>& fb,
                        const std::vector<int64_t>& off, double* out) {
  bool direct = false;
  for (const FarBlock& f : fb) direct |= f.direct && f.rank > 0;
  if (direct && !c->eye_ready) {  // the identity C of directly output factors
    const int64_t ne = int64_t(EYE_LD) * EYE_LD;
    c->own[BUF_EYE].ensure(size_t(ne));
    eye_kernel<<<int((ne + 255) / 256), 256, 0, c->s>>>(c->own[BUF_EYE].p, ne, EYE_LD);
    CK(cudaGetLastError());
    c->launches++;
    c->eye_ready = true;
  }
  std::vector<SmallJob> jl;
  int rows_max = 1;
  for (size_t i = 0; i < fb.size(); ++i) {
    const FarBlock& f = fb[i];
    if (f.rank == 0) continue;
    double* left = out + off[i];
    double* right = left + int64_t(f.m) * f.rank;
    if (f.direct) {  // matrix-free factors as produced (C = identity)
      if (f.rank > EYE_LD) throw hx::Unsupported("factor rank above the identity operand");
      jl.push_back(SmallJob{f.Y, c->buf(BUF_EYE), nullptr, left, f.m, f.rank, EYE_LD, f.m,
                            f.rank});
      jl.push_back(SmallJob{f.Bt, c->buf(BUF_EYE), nullptr, right, f.n, f.rank, EYE_LD, f.n,
                            f.rank});
    } else if (f.dense) {
      jl.push_back(SmallJob{f.Y, f.W, f.sig, left, f.m, f.l, f.l, f.m, f.rank});
      jl.push_back(SmallJob{nullptr, f.V, nullptr, right, f.n, f.l, f.l, 0, f.rank});
    } else {
      jl.push_back(SmallJob{f.Y, f.V, f.sig, left, f.m, f.l, f.l, f.m, f.rank});
      jl.push_back(SmallJob{f.Bt, f.W, nullptr, right, f.n, f.l, f.l, f.n, f.rank});
    }
    rows_max = std::max(rows_max, std::max(f.m, f.n));
  }
  if (!jl.empty()) {
    c->small_jobs.upload(jl, c->s);
    dim3 grid(unsigned(jl.size()), unsigned(std::min(8, (rows_max + 127) / 128)));
    small_product_kernel<<<grid, 128, 0, c->s>>>(c->small_jobs.p);
    CK(cudaGetLastError());
    c->launches++;
  }
}

}  // namespace

#include "traditional_exec.cuh"

extern "C" int hx_ctx_create(int device, hx_ctx** out) {
  return guarded([&]() -> int {
    if (!out) return fail(HX_EINVAL, "null out");
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) return fail(HX_EINVAL, "no such CUDA device");
    CK(cudaSetDevice(device));
    auto* c = new hx_ctx();
    c->device = device;
    CK(cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->s2, cudaStreamNonBlocking));
    int lo_prio = 0, hi_prio = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    CK(cudaStreamCreateWithPriority(&c->s_hi, cudaStreamNonBlocking, hi_prio));
    CK(cudaStreamCreateWithFlags(&c->s3, cudaStreamNonBlocking));
    for (auto& e : c->ev) CK(cudaEventCreate(&e));
    CK(cudaEventCreateWithFlags(&c->up_ev, cudaEventDisableTiming));
    *out = c;
    return HX_OK;
  });
}

extern "C" int hx_ctx_operand(hx_ctx* c, int which, const double* host, const double* device,
                              int64_t n) {
  return guarded([&]() -> int {
    if (!c || which < 0 || which > 1 || n < 0) return fail(HX_EINVAL, "bad operand arguments");
    CK(cudaSetDevice(c->device));
    if (which == 1) c->alias = false;
    if (host) {
      c->attached[which] = nullptr;
      c->own[which].ensure(size_t(n));
      CK(cudaMemcpyAsync(c->own[which].p, host, size_t(n) * sizeof(double),
                         cudaMemcpyHostToDevice, c->s));
      CK(cudaEventRecord(c->up_ev, c->s));  // contexts sharing the pool wait on this
    } else if (device) {
      c->attached[which] = const_cast<double*>(device);
    } else {
      return fail(HX_EINVAL, "need a host or a device pool");
    }
    c->opnd_elems[which] = n;
    return HX_OK;
  });
}

extern "C" int hx_ctx_operand_share(hx_ctx* dst, hx_ctx* src) {
  return guarded([&]() -> int {
    if (!dst || !src || dst == src) return fail(HX_EINVAL, "bad contexts");
    if (dst->device != src->device) return fail(HX_EINVAL, "contexts on different devices");
    if (!src->buf(BUF_A) || !src->buf(BUF_B)) return fail(HX_EINVAL, "source operands not set");
    // host-copied pools: the sharing context's stream waits for the upload on the device,
    // so the host goes on planning the first chunks while the pools are in flight
    CK(cudaStreamWaitEvent(dst->s, src->up_ev, 0));
    dst->attached[0] = src->buf(BUF_A);
    dst->opnd_elems[0] = src->opnd_elems[0];
    dst->alias = src->alias;
    dst->attached[1] = src->alias ? nullptr : src->buf(BUF_B);
    dst->opnd_elems[1] = src->opnd_elems[1];
    return HX_OK;
  });
}

extern "C" int hx_ctx_reset_hints(hx_ctx* c) {
  if (!c) return fail(HX_EINVAL, "null context");
  std::fill(c->rank_hint, c->rank_hint + 32, -1);
  std::fill(c->class_retry, c->class_retry + 32, int8_t(0));
  std::fill(c->iter_hint, c->iter_hint + 32, -1);
  return HX_OK;
}

extern "C" int hx_ctx_trim(hx_ctx* c) {
  return guarded([&]() -> int {
    if (!c) return fail(HX_EINVAL, "null ctx");
    CK(cudaSetDevice(c->device));
    CK(cudaStreamSynchronize(c->s));
    CK(cudaStreamSynchronize(c->s2));
    for (int i = BUF_TERM; i < NUM_BUFS; ++i) {
      if (i == BUF_WORK) {  // points into work[] (released below)
        c->own[i].p = nullptr;
        c->own[i].cap = 0;
        continue;
      }
      c->own[i].release();
    }
    for (int i = 0; i < 3; ++i) {
      c->terms[i].release();
      c->tiles[i].release();
      c->groups[i].release();
    }
    c->sumsq.release();
    c->fro2.release();
    c->seg_b.release();
    c->seg_e.release();
    c->gcols.release();
    c->rterms.release();
    c->rtiles.release();
    c->rgroups.release();
    c->xterms.release();
    c->xtiles.release();
    c->xgroups.release();
    c->gtiles.release();
    c->gsegs.release();
    c->esum.release();
    c->est.release();
    c->qr_jobs.release();
    c->jac_jobs.release();
    c->sel_jobs.release();
    c->small_jobs.release();
    c->rank_d.release();
    c->retry_d.release();
    c->rsum.release();
    c->resid.release();
    c->tb.release();
    c->te.release();
    for (auto& w : c->work) w.release();
    c->trad_release(true);
    c->omega_rows = 0;
    c->omega_cols = 0;
    c->omega_seed = ~0ULL;
    c->eye_ready = false;
    c->trans_recs.release();
    c->out_far = c->near_begin = c->near_elems = 0;
    c->res_rank.clear();
    c->res_deg.clear();
    c->res_off.clear();
    return HX_OK;
  });
}

extern "C" int hx_ctx_operand_alias(hx_ctx* c) {
  if (!c) return fail(HX_EINVAL, "null ctx");
  c->alias = true;
  c->opnd_elems[1] = c->opnd_elems[0];
  return HX_OK;
}

// NVTX ranges over the product phases (visible in Nsight timelines; no-ops without a tool)
struct NvtxPhases {
  bool open = false;
  void next(const char* name) {
    if (open) nvtxRangePop();
    nvtxRangePushA(name);
    open = true;
  }
  ~NvtxPhases() {
    if (open) nvtxRangePop();
  }
};

// HX_RECOMP_TIMING: synchronizing wall-clock marks through the recompression phase (a
// diagnostic: it serializes host list building and device work)
struct PhaseMarks {
  bool on = std::getenv("HX_RECOMP_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  std::vector<std::pair<std::string, double>> acc;
  void mark(const char* what, cudaStream_t s) {
    if (!on) return;
    CK(cudaStreamSynchronize(s));
    const auto now = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(now - t).count();
    t = now;
    for (auto& a : acc)
      if (a.first == what) { a.second += ms; return; }
    acc.emplace_back(what, ms);
  }
  ~PhaseMarks() {
    if (!on) return;
    for (auto& a : acc) std::fprintf(stderr, "[hx recomp] %-14s %9.1f ms\n", a.first.c_str(), a.second);
  }
};

extern "C" int hx_product(hx_ctx* c, hx_plan* P, const hx_product_cfg* cfg,
                          hx_product_stats* st) {
  return guarded([&]() -> int {
    if (!c || !P || !cfg) return fail(HX_EINVAL, "null argument");
    if (cfg->policy == 0 && !(cfg->eps > 0.0)) return fail(HX_EINVAL, "eps must be positive");
    if (cfg->policy == 1 && cfg->k_max < 1) return fail(HX_EINVAL, "k_max must be >= 1");
    if (!c->buf(BUF_A) || !c->buf(BUF_B)) return fail(HX_EINVAL, "operands not set");
    CK(cudaSetDevice(c->device));
    const int over = cfg->oversample > 0 ? cfg->oversample : 6;
    HostMarks hm(c);
    NvtxPhases nvtx;
    nvtx.next("hx::setup");
    c->launches = 0;
    {
      const double key[4] = {double(cfg->policy), cfg->eps, double(cfg->k_max), double(cfg->tag)};
      if (!std::equal(key, key + 4, c->hint_key)) {
        std::copy(key, key + 4, c->hint_key);
        std::fill(c->rank_hint, c->rank_hint + 32, -1);
        std::fill(c->class_retry, c->class_retry + 32, int8_t(0));
        std::fill(c->iter_hint, c->iter_hint + 32, -1);
      }
    }
    static const bool use_hints = std::getenv("HX_NO_RANK_HINT") == nullptr;
    cudaStream_t s = c->s;
    CK(cudaEventRecord(c->ev[0], s));

    // ---- buffers: every size is known before the factor work lists are filled
    c->own[BUF_CORE].ensure(size_t(P->core_elems));
    c->own[BUF_TERM].ensure(size_t(P->term_elems));
    c->own[BUF_TILE].ensure(size_t(P->tile_elems));
    c->sumsq.ensure(size_t(P->n_sumsq));
    for (int i = 0; i < 2; ++i) {
      c->terms[i].ensure(i ? P->fac_terms.size() : P->core_terms.size());
      c->tiles[i].ensure(i ? P->fac_tiles.size() : P->core_tiles.size());
      c->groups[i].ensure(i ? P->fac_groups.size() : P->core_groups.size());
    }
    c->terms[2].ensure(P->mat_terms.size());
    c->tiles[2].ensure(P->mat_tiles.size());
    c->groups[2].ensure(P->mat_groups.size());
    c->gcols.ensure(P->gcols.size());
    // column records first on the compute stream; the materialization lists on the copy
    // stream, overlapping the whole formation phase (host arrays are page-locked)
    auto h2d = [](void* d, const void* h, size_t bytes, cudaStream_t st) {
      if (bytes) CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
    };
    h2d(c->gcols.p, P->gcols.data(), P->gcols.size() * sizeof(ColRec), s);
    // ragged trees: identity operand and transposed dense blocks of H-block x dense terms
    if (P->needs_eye && !c->eye_ready) {
      const int64_t ne = int64_t(EYE_LD) * EYE_LD;
      c->own[BUF_EYE].ensure(size_t(ne));
      eye_kernel<<<int((ne + 255) / 256), 256, 0, s>>>(c->own[BUF_EYE].p, ne, EYE_LD);
      CK(cudaGetLastError());
      c->launches++;
      c->eye_ready = true;
    }
    if (!P->dtrans.empty()) {
      c->own[BUF_GATHER].ensure(size_t(P->dtrans_elems));
      c->trans_recs.upload(P->dtrans, s);
      transpose_kernel<<<int(P->dtrans.size()), 256, 0, s>>>(c->trans_recs.p, c->buf(BUF_A),
                                                             c->own[BUF_GATHER].p);
      CK(cudaGetLastError());
      c->launches++;
    }
    CK(cudaEventRecord(c->ev[6], s));
    CK(cudaStreamWaitEvent(c->s2, c->ev[6], 0));  // buffers allocated before s2 copies
    h2d(c->terms[2].p, P->mat_terms.data(), P->mat_terms.size() * sizeof(Term), c->s2);
    h2d(c->tiles[2].p, P->mat_tiles.data(), P->mat_tiles.size() * sizeof(Tile), c->s2);
    h2d(c->groups[2].p, P->mat_groups.data(), P->mat_groups.size() * sizeof(Group), c->s2);
    CK(cudaEventRecord(c->ev[7], c->s2));
    BufPtrs bp = c->ptrs();
    CK(cudaEventRecord(c->ev[5], s));

    nvtx.next("hx::form");
    // ---- 1. term formation: gather thin factors per X-group, cores, X G products.
    // Deferred plans fill each batch's work lists here, on the host, while the device
    // runs the previous batch.
    // Consecutive batches are independent (different X-groups): odd batches run on a
    // second stream with their own copy of the core workspace, so one batch's X G bands
    // overlap the next batch's cores.
    const bool two = P->batches.size() > 1 && !std::getenv("HX_ONE_FORM_STREAM");
    BufPtrs bp_odd = bp;
    if (two) {
      c->own[BUF_CORE].ensure(size_t(2 * P->core_elems));
      bp = c->ptrs();
      bp_odd = bp;
      bp_odd.p[BUF_CORE] = bp.p[BUF_CORE] + P->core_elems;
      CK(cudaEventRecord(c->ev[6], s));
      CK(cudaStreamWaitEvent(c->s3, c->ev[6], 0));
    }
    for (size_t bi = 0; bi < P->batches.size(); ++bi) {
      if (!P->batch_ready[bi]) {
        P->fill_batch(int64_t(bi));
        P->batch_ready[bi] = 1;
      }
      const hx_plan::Batch& bt = P->batches[bi];
      const bool odd = two && (bi & 1);
      const cudaStream_t fs = odd ? c->s3 : s;
      const BufPtrs& fbp = odd ? bp_odd : bp;
      h2d(c->tiles[0].p + bt.core_begin, P->core_tiles.data() + bt.core_begin,
          size_t(bt.core_end - bt.core_begin) * sizeof(Tile), fs);
      h2d(c->groups[0].p + bt.cg_begin, P->core_groups.data() + bt.cg_begin,
          size_t(bt.cg_end - bt.cg_begin) * sizeof(Group), fs);
      h2d(c->terms[0].p + bt.cm_begin, P->core_terms.data() + bt.cm_begin,
          size_t(bt.cm_end - bt.cm_begin) * sizeof(Term), fs);
      h2d(c->tiles[1].p + bt.fac_begin, P->fac_tiles.data() + bt.fac_begin,
          size_t(bt.fac_end - bt.fac_begin) * sizeof(Tile), fs);
      h2d(c->groups[1].p + bt.fg_begin, P->fac_groups.data() + bt.fg_begin,
          size_t(bt.fg_end - bt.fg_begin) * sizeof(Group), fs);
      h2d(c->terms[1].p + bt.fm_begin, P->fac_terms.data() + bt.fm_begin,
          size_t(bt.fm_end - bt.fm_begin) * sizeof(Term), fs);
      launch_gemm(c, P->tile, c->tiles[0].p + bt.core_begin, c->groups[0].p, c->terms[0].p,
                  int(bt.core_end - bt.core_begin), fbp, nullptr, c->gcols.p, true, fs);
      launch_gemm(c, P->tile, c->tiles[1].p + bt.fac_begin, c->groups[1].p, c->terms[1].p,
                  int(bt.fac_end - bt.fac_begin), fbp, nullptr, c->gcols.p, true, fs);
    }
    if (two) {
      CK(cudaEventRecord(c->ev[6], c->s3));
      CK(cudaStreamWaitEvent(s, c->ev[6], 0));
    }
    CK(cudaEventRecord(c->ev[1], s));
    hm.mark("form-issued");
    nvtx.next("hx::materialize");
    // ---- 2. materialization
    CK(cudaStreamWaitEvent(s, c->ev[7], 0));
    launch_gemm(c, P->tile, c->tiles[2].p, c->groups[2].p, c->terms[2].p,
                int(P->mat_tiles.size()), bp, c->sumsq.p);
    CK(cudaEventRecord(c->ev[2], s));

    // ---- per-leaf squared Frobenius norms
    const int nl = int(P->leaves.size());
    std::vector<int> sb(nl), se(nl);
    for (int i = 0; i < nl; ++i) {
      sb[i] = P->leaves[i].sumsq_begin;
      se[i] = P->leaves[i].sumsq_end;
    }
    c->seg_b.upload(sb, s);
    c->seg_e.upload(se, s);
    c->fro2.ensure(size_t(std::max(nl, 1)));
    if (nl) {
      segment_sum_kernel<<<(nl + 255) / 256, 256, 0, s>>>(c->sumsq.p, c->seg_b.p, c->seg_e.p,
                                                          c->fro2.p, nl);
      CK(cudaGetLastError());
      c->launches++;
    }

    hm.mark("mat-issued");
    nvtx.next("hx::recompress");
    // ---- 3. recompression of far leaves, on the high-priority stream
    const cudaStream_t s_main = s;
    CK(cudaEventRecord(c->ev[6], s));
    CK(cudaStreamWaitEvent(c->s_hi, c->ev[6], 0));
    s = c->s_hi;
    c->s = s;
    struct RestoreStream {
      hx_ctx* c;
      cudaStream_t s;
      ~RestoreStream() { c->s = s; }
    } restore_stream{c, s_main};
    PhaseMarks pm;
    pm.mark("materialize", s);
    std::vector<FarBlock> fb;
    int mu_max = 0;
    for (int i = 0; i < nl; ++i) {
      const OutLeaf& L = P->leaves[i];
      if (L.kind != 1) continue;
      FarBlock f;
      f.leaf = i;
      f.m = L.m;
      f.n = L.n;
      f.mu = std::min(L.m, L.n);
      f.t_off = L.ws_off;
      f.fro2 = c->fro2.p + i;
      fb.push_back(f);
      mu_max = std::max(mu_max, f.mu);
    }
    int64_t nmax = 1;
    for (const FarBlock& f : fb) nmax = std::max<int64_t>(nmax, f.n);
    const int lcap = JAC_QMAX;
    if (cfg->tag == 3 &&
        (c->omega_rows < nmax || c->omega_cols < lcap || c->omega_seed != cfg->seed)) {
      c->omega_rows = std::max<int64_t>(nmax, c->omega_rows);
      c->omega_cols = lcap;
      c->omega_seed = cfg->seed;
      const int64_t ne = c->omega_rows * c->omega_cols;
      c->own[BUF_OMEGA].ensure(size_t(ne));
      omega_kernel<<<int((ne + 255) / 256), 256, 0, s>>>(c->own[BUF_OMEGA].p, ne, cfg->seed);
      CK(cudaGetLastError());
      c->launches++;
    }
    // implicit-route leaves: their terms clipped to the leaf; Z rows ordered by column range
    // (factor pairs first), W rows by row range, so that each gathered tile shares one range
    int64_t zmax = 0;
    std::vector<int> impl_idx;
    for (int i = 0; i < int(fb.size()); ++i)
      if (P->leaves[fb[size_t(i)].leaf].implicit) impl_idx.push_back(i);
    par_for(int(impl_idx.size()), [&](int q) {
      FarBlock& f = fb[size_t(impl_idx[size_t(q)])];
      const OutLeaf& L = P->leaves[f.leaf];
      f.implicit = 1;
      for (int32_t g = L.g_begin; g < L.g_end; ++g) {
        const Group gr = P->mat_groups[g];
        for (int32_t ti = gr.t_begin; ti < gr.t_end; ++ti) {
          const Term& tm = P->mat_terms[ti];
          if (tm.k <= 0) continue;
          ImplTerm x;
          x.t = tm;
          x.k = tm.k;
          x.lr = (tm.a_kc == 0 && tm.b_kc == 0) ? 1 : 0;
          const int64_t r0 = std::max<int64_t>(tm.r_lo, L.row0);
          const int64_t r1 = std::min<int64_t>(int64_t(tm.r_lo) + tm.rows, L.row0 + L.m);
          const int64_t c0 = std::max<int64_t>(tm.c_lo, L.col0);
          const int64_t c1 = std::min<int64_t>(int64_t(tm.c_lo) + tm.cols, L.col0 + L.n);
          if (r1 <= r0 || c1 <= c0) continue;
          x.ri = int(r0 - L.row0);
          x.rn = int(r1 - r0);
          x.ci = int(c0 - L.col0);
          x.cn = int(c1 - c0);
          f.it.push_back(x);
        }
      }
      std::vector<int> o(f.it.size());
      for (size_t i = 0; i < o.size(); ++i) o[i] = int(i);
      std::stable_sort(o.begin(), o.end(), [&](int a, int b) {
        const ImplTerm &x = f.it[a], &y = f.it[b];
        if (x.lr != y.lr) return x.lr > y.lr;
        if (x.ci != y.ci) return x.ci < y.ci;
        return x.cn < y.cn;
      });
      // rows of each term start at an even row (16-byte aligned k-contiguous reads)
      int64_t r = 0;
      for (int i : o) {
        f.it[i].zrow = r;
        r = (r + f.it[i].k + 1) & ~int64_t(1);
      }
      f.zrows = r;
      f.zorder = o;
      std::stable_sort(o.begin(), o.end(), [&](int a, int b) {
        const ImplTerm &x = f.it[a], &y = f.it[b];
        if (x.lr != y.lr) return x.lr > y.lr;
        if (x.ri != y.ri) return x.ri < y.ri;
        return x.rn < y.rn;
      });
      r = 0;
      for (int i : o) {
        f.it[i].wrow = r;
        r = (r + f.it[i].k + 1) & ~int64_t(1);
      }
      f.worder = o;
    });
    (void)zmax;
    if (std::getenv("HX_IMPL_STATS")) {
      double full = 0, part = 0, part_area = 0, dd = 0, nl_impl = 0, full_terms = 0, part_terms = 0;
      for (const FarBlock& f : fb) {
        if (!f.implicit) continue;
        nl_impl += 1;
        for (const ImplTerm& x : f.it) {
          if (!x.lr) { dd += x.k; continue; }
          if (x.rn == f.m && x.cn == f.n) { full += x.k; full_terms += 1; }
          else { part += x.k; part_area += double(x.k) * x.rn * x.cn; part_terms += 1; }
        }
      }
      std::fprintf(stderr, "[hx impl] leaves %.0f: full-range rows %.0f (%.0f terms), partial rows "
                   "%.0f (%.0f terms, mean area %.0f), dxd rows %.0f\n", nl_impl, full, full_terms,
                   part, part_terms, part > 0 ? part_area / part : 0.0, dd);
    }

    // Rows of one gathered operand (segments in output-row order, kb / ke in B-row
    // coordinates) packed into tiles of 64 consecutive output rows; a tile's K range is the
    // union of its rows' ranges (rows are zero-filled outside their own).
    auto gather_rows = [](GatherSet& gs, const std::vector<GSeg>& sg, uint8_t out_buf,
                          int64_t out_off, int32_t out_ld, uint8_t b_buf, int64_t b_base,
                          int32_t b_ld, int C) {
      std::vector<GSeg> cur;
      int rows = 0;
      int64_t row_base = 0;
      int kmin = 1 << 30, kmax = 0;
      auto flush = [&]() {
        if (!rows) return;
        if (kmax <= kmin) kmin = kmax = 0;  // pad rows only
        for (GSeg& x : cur) {
          x.kb -= kmin;
          x.ke -= kmin;
        }
        for (int j = 0; j < C; j += 64) {
          GTile t;
          std::memset(&t, 0, sizeof(t));
          t.out_off = out_off + row_base + int64_t(j) * out_ld;
          t.out_ld = out_ld;
          t.b_off = b_base + kmin + int64_t(j) * b_ld;
          t.b_ld = b_ld;
          t.seg_begin = int32_t(gs.segs.size());
          gs.segs.insert(gs.segs.end(), cur.begin(), cur.end());
          t.seg_end = int32_t(gs.segs.size());
          t.klen = kmax - kmin;
          t.rows = int16_t(rows);
          t.cols = int16_t(std::min(64, C - j));
          t.out_buf = out_buf;
          t.b_buf = b_buf;
          gs.tiles.push_back(t);
        }
        row_base += rows;
        rows = 0;
        kmin = 1 << 30;
        kmax = 0;
        cur.clear();
      };
      for (GSeg x : sg) {
        while (x.rows > 0) {
          const int n = std::min<int>(x.rows, 64 - rows);
          GSeg part = x;
          part.rows = int16_t(n);
          cur.push_back(part);
          if (x.ke > x.kb) {  // pad segments (kb == ke) only write zero rows
            kmin = std::min(kmin, x.kb);
            kmax = std::max(kmax, x.ke);
          }
          rows += n;
          x.off += int64_t(n) * x.ld;
          x.rows = int16_t(x.rows - n);
          if (rows == 64) flush();
        }
      }
      flush();
    };

    pm.mark("impl-lists", s);
    constexpr int PR = 8;  // probe columns of the implicit route's tail estimate
    // Jacobi on R^T (rows of the QR factor): fewer sweeps than on the columns of R
    const char* jt = std::getenv("HX_JAC_TRANS");
    const int jac_trans = jt ? std::atoi(jt) : 1;
    int64_t matvecs = 0;  // the reference's CountingMap total (compressors.py:88-119)
    int64_t sketch_cols = 0;  // operator columns the sketch route actually applied
    int rounds = 0;
    std::vector<int> active;
    const bool iterative = cfg->tag >= 0 && cfg->tag <= 2 && !P->trad;
    if (P->trad) {
      hm.mark("iter-start");
      matvecs = run_traditional(c, P, cfg, fb, rounds);
      hm.mark("iter-done");
    } else if (iterative) {
      hm.mark("iter-start");
      matvecs = recompress_iterative(c, P, cfg, fb, jac_trans, rounds);
      hm.mark("iter-done");
    } else {
      for (int i = 0; i < int(fb.size()); ++i) active.push_back(i);
      // dense-svd materializes S I (apply_mat of the identity): n columns per block
      for (const FarBlock& f : fb) matvecs += f.n;
    }
    const bool explicit_tail = cfg->policy == 0 && cfg->eps < 1e-6;
    while (!active.empty()) {
      if (rounds >= 6) throw std::runtime_error("sketch adaptation did not converge");
      auto a16 = [](int64_t x) { return (x + 15) & ~int64_t(15); };
      // sketch widths for this round
      int64_t wsz = 0, zsz = 0;
      for (int i : active) {
        FarBlock& f = fb[i];
        int l;
        if (cfg->policy == 1) {
          l = std::min(f.mu, cfg->k_max + over);
        } else if (f.l == 0) {
          l = cfg->sketch0 > 0 ? cfg->sketch0 : default_sketch(f.mu);
          const int h = c->rank_hint[ilog2(f.mu)];
          // narrowed only when the saving is large (a hint that undershoots costs a retry);
          // widened when blocks of this class needed a retry before (config 5's 128-blocks:
          // ranks up to 19 against a 24-column default sketch)
          const int lh = std::max(16, (h + over + 8 + 7) & ~7);
          if (cfg->sketch0 <= 0 && h >= 0 && use_hints) {
            if (c->class_retry[ilog2(f.mu)]) l = std::max(l, lh);
            else if (4 * lh <= 3 * l) l = lh;
          }
        } else {
          l = 2 * f.l;
        }
        l = std::min(l, f.mu);
        const int cap = f.implicit ? lcap - PR : lcap;
        if (l > cap) {
          if (f.mu <= cap) l = f.mu;
          else throw hx::Unsupported("block needs a sketch wider than " + std::to_string(cap));
        }
        f.l = l;
        f.dense = (!f.implicit && f.m >= f.n && l == f.n) ? 1 : 0;
        f.round = rounds;
        const int64_t q = l;
        if (f.implicit) {
          wsz += a16(int64_t(f.m) * (q + PR)) + a16(int64_t(f.n) * q) + a16(q * PR);
          f.zoff = zsz;
          zsz += a16(f.zrows * (q + PR));
        } else if (!f.dense) {
          wsz += a16(int64_t(f.m) * q) + a16(int64_t(f.n) * q);
        }
        wsz += 3 * a16(q * q) + a16(q);
      }
      if (int(c->work.size()) <= rounds) c->work.resize(rounds + 1);
      c->work[rounds].ensure(size_t(std::max<int64_t>(wsz, 16)));
      double* wb = c->work[rounds].p;
      c->own[BUF_WORK].p = wb;  // buffer id BUF_WORK points at this round's workspace
      if (zsz > 0) c->own[BUF_CORE].ensure(size_t(zsz));  // Z / W blocks (cores are dead)
      bp = c->ptrs();
      int64_t pos = 0;
      auto take = [&](int64_t nelem) {
        double* p = wb + pos;
        pos += a16(nelem);
        return p;
      };
      auto woff = [&](const double* p) { return int64_t(p - wb); };
      pm.mark("l-widths", s);
      // every work list of the round is known up front: one upload, then launches in order
      GemmSet gm;
      GatherSet ga;
      std::vector<QrJob> qy, qb;
      std::vector<int> tail_b, tail_e, est_b, est_e;
      int tail_slots = 0, est_slots = 0;
      // -- batch 0 / gather 0: Z = R^T Omega of the implicit leaves
      for (int i : active) {
        FarBlock& f = fb[i];
        const int l = f.l;
        if (f.dense) {
          f.Y = c->buf(BUF_TILE) + f.t_off;  // QR in place of the materialized block
          f.Bt = nullptr;
        } else if (f.implicit) {
          f.Y = take(int64_t(f.m) * (l + PR));
          f.Bt = take(int64_t(f.n) * l);
          f.C1 = take(int64_t(l) * PR);
        } else {
          f.Y = take(int64_t(f.m) * l);
          f.Bt = take(int64_t(f.n) * l);
        }
        f.R = take(int64_t(l) * l);
        f.W = take(int64_t(l) * l);
        f.V = take(int64_t(l) * l);
        f.sig = take(l);
        if (f.implicit) sketch_cols += 2 * (l + PR);
        else if (f.dense) sketch_cols += f.n;
        else sketch_cols += 2 * l;
      }
      par_build(active, gm, ga, [&](int i, GemmSet& gm, GatherSet& ga) {
        FarBlock& f = fb[i];
        const int l = f.l;
        if (!f.implicit) return;
        const OutLeaf& L = P->leaves[f.leaf];
        const int Lw = l + PR;
        std::vector<GSeg> run;
        int64_t have = 0;  // rows covered so far (pad segments fill the alignment gaps)
        for (int q : f.zorder) {  // ascending Z rows
          const ImplTerm& x = f.it[q];
          const Term& tm = x.t;
          const int64_t jo = L.col0 + x.ci - tm.c_lo;  // first leaf column, term-local
          if (x.lr) {
            if (x.zrow > have)
              run.push_back(GSeg{tm.b_off, 0, int16_t(x.zrow - have), tm.b_buf, 0, 0, 0});
            have = x.zrow + x.k;
            run.push_back(GSeg{tm.b_off + jo, tm.b_ld, int16_t(x.k), tm.b_buf, 0, x.ci,
                               x.ci + x.cn});
          } else {
            // dense x dense: Z_t = D_B[:, cols] Omega[cols, :]
            const Term z = mk(tm.b_buf, tm.b_off + jo * tm.b_ld, tm.b_ld, 0, BUF_OMEGA, x.ci,
                              int32_t(c->omega_rows), 1, x.cn, x.k, Lw);
            const int32_t g = gm.group(&z, 1);
            gm.cover(g, BUF_CORE, f.zoff + x.zrow, int32_t(f.zrows), x.k, Lw, 0, 0);
          }
        }
        gather_rows(ga, run, BUF_CORE, f.zoff, int32_t(f.zrows), BUF_OMEGA, 0,
                    int32_t(c->omega_rows), Lw);
      });
      gm.cut();  // gemm batch 0
      ga.cut();  // gather batch 0
      pm.mark("l-b0", s);
      // -- batch 1: Y = T Omega (materialized) / Y = sum L_t Z_t (implicit)
      for (int i : active) {
        const FarBlock& f = fb[i];
        qy.push_back(QrJob{f.Y, f.R, f.m, f.dense ? f.n : f.l});
      }
      par_build(active, gm, ga, [&](int i, GemmSet& gm, GatherSet&) {
        FarBlock& f = fb[i];
        const int l = f.l;
        if (f.dense) {
          return;
        } else if (f.implicit) {
          const OutLeaf& L = P->leaves[f.leaf];
          std::vector<Term> ts;
          std::vector<std::pair<int, int>> band;
          ts.reserve(f.it.size() + size_t(L.tsub_end - L.tsub_begin));
          band.reserve(f.it.size() + size_t(L.tsub_end - L.tsub_begin));
          for (int q : f.worder) {  // (lr, row band): terms sharing a band are adjacent
            const ImplTerm& x = f.it[size_t(q)];
            Term y = mk(x.t.a_buf, x.t.a_off, x.t.a_ld, x.t.a_kc, BUF_CORE, f.zoff + x.zrow,
                        int32_t(f.zrows), 1, x.k, x.t.rows, l + PR);
            y.r_lo = x.t.r_lo;
            ts.push_back(y);
            band.emplace_back(x.ri, x.rn);
          }
          for (int32_t q = L.tsub_begin; q < L.tsub_end; ++q) {
            // + T_sub Omega: one term per dense block of the block-sparse T_sub
            const TSubBlock& tb = P->tsub[size_t(q)];
            Term y = mk(BUF_TILE, tb.off, tb.h, 0, BUF_OMEGA, tb.c0 - L.col0,
                        int32_t(c->omega_rows), 1, tb.w, tb.h, l + PR);
            y.r_lo = int32_t(tb.r0);
            ts.push_back(y);
            band.emplace_back(int(tb.r0 - L.row0), tb.h);
          }
          gm.cover_banded(ts, band, BUF_WORK, woff(f.Y), f.m, f.m, l + PR, int(L.row0), 0, true);
        } else {
          const Term y = mk(BUF_TILE, f.t_off, f.m, 0, BUF_OMEGA, 0, int32_t(c->omega_rows), 1,
                            f.n, f.m, l);
          const int32_t g = gm.group(&y, 1);
          gm.cover(g, BUF_WORK, woff(f.Y), f.m, f.m, l, 0, 0);
        }
      });
      gm.cut();  // gemm batch 1
      pm.mark("l-b1", s);
      // -- batches 2, 3 (implicit): C1 = Q^T Y_probe; ||Y_probe - Q C1||^2 per tile
      for (int i : active) {
        FarBlock& f = fb[i];
        if (f.implicit) {
          const int l = f.l;
          const Term t1 = mk(BUF_WORK, woff(f.Y), f.m, 1, BUF_WORK, woff(f.Y) + int64_t(f.m) * l,
                             f.m, 1, f.m, l, PR);
          const int32_t g = gm.group(&t1, 1);
          gm.cover(g, BUF_WORK, woff(f.C1), l, l, PR, 0, 0);
        }
      }
      gm.cut();  // gemm batch 2
      for (size_t a = 0; a < active.size(); ++a) {
        FarBlock& f = fb[active[a]];
        est_b.push_back(est_slots);
        if (f.implicit) {
          const int l = f.l;
          const Term t2 = mk(BUF_WORK, woff(f.Y), f.m, 0, BUF_WORK, woff(f.C1), l, 1, l, f.m, PR);
          const int32_t g = gm.group(&t2, 1);
          gm.cover(g, BUF_WORK, woff(f.Y) + int64_t(f.m) * l, f.m, f.m, PR, 0, 0,
                   MODE_RESID_SUMSQ, &est_slots);
        }
        est_e.push_back(est_slots);
      }
      gm.cut();  // gemm batch 3
      pm.mark("l-b23", s);
      // -- gather 1 + batch 4: W = L^T Q (implicit), rows sharing a row range
      par_build(active, gm, ga, [&](int i, GemmSet& gm, GatherSet& ga) {
        FarBlock& f = fb[i];
        if (!f.implicit) return;
        const OutLeaf& L = P->leaves[f.leaf];
        const int l = f.l;
        std::vector<GSeg> run;
        int64_t have = 0;  // rows covered so far (pad segments fill the alignment gaps)
        for (int q : f.worder) {  // ascending W rows
          const ImplTerm& x = f.it[q];
          const Term& tm = x.t;
          const int64_t io = L.row0 + x.ri - tm.r_lo;  // first leaf row, term-local
          if (x.lr) {
            if (x.wrow > have)
              run.push_back(GSeg{tm.a_off, 0, int16_t(x.wrow - have), tm.a_buf, 0, 0, 0});
            have = x.wrow + x.k;
            run.push_back(GSeg{tm.a_off + io, tm.a_ld, int16_t(x.k), tm.a_buf, 0, x.ri,
                               x.ri + x.rn});
          } else {
            // dense x dense: W_t = D_A[rows, :]^T Q[rows, :]
            const Term w = mk(tm.a_buf, tm.a_off + io, tm.a_ld, 1, BUF_WORK, woff(f.Y) + x.ri,
                              f.m, 1, x.rn, x.k, l);
            const int32_t g = gm.group(&w, 1);
            gm.cover(g, BUF_CORE, f.zoff + x.wrow, int32_t(f.zrows), x.k, l, 0, 0);
          }
        }
        gather_rows(ga, run, BUF_CORE, f.zoff, int32_t(f.zrows), BUF_WORK, woff(f.Y), f.m, l);
      });
      gm.cut();  // gemm batch 4
      ga.cut();  // gather batch 1
      pm.mark("l-b4", s);
      // -- batch 5: Bt = T^T Q (materialized) / Bt = sum R_t W_t (implicit)
      for (int i : active) {
        const FarBlock& f = fb[i];
        if (!f.dense) qb.push_back(QrJob{f.Bt, f.R, f.n, f.l});
      }
      par_build(active, gm, ga, [&](int i, GemmSet& gm, GatherSet&) {
        FarBlock& f = fb[i];
        if (f.dense) return;
        const int l = f.l;
        if (f.implicit) {
          const OutLeaf& L = P->leaves[f.leaf];
          std::vector<Term> ts;
          std::vector<std::pair<int, int>> band;
          ts.reserve(f.it.size() + 1);
          band.reserve(f.it.size() + 1);
          for (int q : f.zorder) {  // (lr, column band): terms sharing a band are adjacent
            const ImplTerm& x = f.it[size_t(q)];
            // R_t(j, kk) = Q_t(kk, j)
            Term y = mk(x.t.b_buf, x.t.b_off, x.t.b_ld, uint8_t(x.t.b_kc ? 1 : 0), BUF_CORE,
                        f.zoff + x.wrow, int32_t(f.zrows), 1, x.k, x.t.cols, l);
            y.r_lo = x.t.c_lo;
            ts.push_back(y);
            band.emplace_back(x.ci, x.cn);
          }
          for (int32_t q = L.tsub_begin; q < L.tsub_end; ++q) {  // + T_sub^T Q, block by block
            const TSubBlock& tb = P->tsub[size_t(q)];
            Term y = mk(BUF_TILE, tb.off, tb.h, 1, BUF_WORK, woff(f.Y) + (tb.r0 - L.row0), f.m, 1,
                        tb.h, tb.w, l);
            y.r_lo = int32_t(tb.c0);
            ts.push_back(y);
            band.emplace_back(int(tb.c0 - L.col0), tb.w);
          }
          gm.cover_banded(ts, band, BUF_WORK, woff(f.Bt), f.n, f.n, l, int(L.col0), 0, true);
        } else {
          const Term y = mk(BUF_TILE, f.t_off, f.m, 1, BUF_WORK, woff(f.Y), f.m, 1, f.m, f.n, l);
          const int32_t g = gm.group(&y, 1);
          gm.cover(g, BUF_WORK, woff(f.Bt), f.n, f.n, l, 0, 0);
        }
      });
      gm.cut();  // gemm batch 5
      pm.mark("l-b5", s);
      // -- batch 6: tight tolerances, materialized blocks: ||T||^2 - sum s_i^2 cancels below
      // ~1e-15 ||T||^2, so the unsampled tail is measured directly as ||T - Q Bt^T||_F^2
      for (int i : active) {
        FarBlock& f = fb[i];
        tail_b.push_back(tail_slots);
        if (explicit_tail && !f.dense && !f.implicit) {
          const Term y = mk(BUF_WORK, woff(f.Y), f.m, 0, BUF_WORK, woff(f.Bt), f.n, 0, f.l, f.m,
                            f.n);
          const int32_t g = gm.group(&y, 1);
          gm.cover(g, BUF_TILE, f.t_off, f.m, f.m, f.n, 0, 0, MODE_RESID_SUMSQ, &tail_slots);
        }
        tail_e.push_back(tail_slots);
      }
      gm.cut();  // gemm batch 6
      pm.mark("host-lists", s);
      // upload and run
      const int na = int(active.size());
      c->xterms.upload(gm.terms, s);
      c->xtiles.upload(gm.tiles, s);
      c->xgroups.upload(gm.groups, s);
      if (!ga.tiles.empty()) {
        c->gtiles.upload(ga.tiles, s);
        c->gsegs.upload(ga.segs, s);
      }
      c->rsum.ensure(size_t(std::max(tail_slots, 1)));
      c->resid.ensure(size_t(std::max(na, 1)));
      c->esum.ensure(size_t(std::max(est_slots, 1)));
      c->est.ensure(size_t(std::max(na, 1)));
      auto gemm_batch = [&](int b, double* sums) {
        const size_t n = gm.count(b);
        static const bool rshort = std::getenv("HX_RSHORT") != nullptr;
        if (n) launch_gemm(c, 64, c->xtiles.p + gm.cuts[size_t(b)], c->xgroups.p, c->xterms.p,
                           int(n), bp, sums, nullptr, rshort);
      };
      auto gather_batch = [&](int b) {
        const size_t n = ga.count(b);
        if (!n) return;
        // warp-specialized persistent kernel unless HX_GATHER_WS=0
        static const bool ws = !(std::getenv("HX_GATHER_WS") && std::getenv("HX_GATHER_WS")[0] == '0');
        static int ggrid = 0;
        if (!ggrid) {
          CK(cudaFuncSetAttribute(gather_gemm_kernel<Gemm64>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, Gemm64::SMEM));
          CK(cudaFuncSetAttribute(gather_gemm_ws_kernel<Ws64>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, Ws64::SMEM));
          int dev = 0, sms = 0, b = 0;
          CK(cudaGetDevice(&dev));
          CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
          CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, gather_gemm_ws_kernel<Ws64>,
                                                           Ws64::THREADS, Ws64::SMEM));
          ggrid = std::max(1, b) * sms;
        }
        if (ws)
          gather_gemm_ws_kernel<Ws64><<<int(std::min<size_t>(n, size_t(ggrid))), Ws64::THREADS,
                                        Ws64::SMEM, s>>>(c->gtiles.p + ga.cuts[size_t(b)],
                                                         c->gsegs.p, bp, int(n));
        else
          gather_gemm_kernel<Gemm64><<<int(n), Gemm64::THREADS, Gemm64::SMEM, s>>>(
              c->gtiles.p + ga.cuts[size_t(b)], c->gsegs.p, bp, int(n));
        CK(cudaGetLastError());
        c->launches++;
      };
      auto seg_sums = [&](const std::vector<int>& b, const std::vector<int>& e, DArr<int>& db,
                          DArr<int>& de, const double* vals, double* out, double scale) {
        db.upload(b, s);
        de.upload(e, s);
        segment_sum_kernel<<<(na + 255) / 256, 256, 0, s>>>(vals, db.p, de.p, out, na, scale);
        CK(cudaGetLastError());
        c->launches++;
      };
      gather_batch(0);
      gemm_batch(0, nullptr);
      gemm_batch(1, nullptr);
      pm.mark("sketch-Y", s);
      run_qr(c, qy);
      if (est_slots) {
        gemm_batch(2, nullptr);
        gemm_batch(3, c->esum.p);
        seg_sums(est_b, est_e, c->eb, c->ee, c->esum.p, c->est.p, 1.0 / PR);
      }
      pm.mark("qr-Y+est", s);
      gather_batch(1);
      gemm_batch(4, nullptr);
      gemm_batch(5, nullptr);
      if (tail_slots) {
        gemm_batch(6, c->rsum.p);
        seg_sums(tail_b, tail_e, c->tb, c->te, c->rsum.p, c->resid.p, 1.0);
      }
      pm.mark("sketch-Bt", s);
      run_qr(c, qb);
      // SVD of the small factor
      std::vector<JacJob> jj;
      for (int i : active) {
        FarBlock& f = fb[i];
        jj.push_back(JacJob{f.R, f.sig, f.W, f.V, f.l, jac_trans});
      }
      if (std::getenv("HX_JAC_STATS")) {
        unsigned long long z[2] = {0, 0};
        CK(cudaStreamSynchronize(s));
        CK(cudaMemcpyToSymbol(g_jac_stats, z, sizeof(z)));
      }
      run_jacobi(c, jj);
      if (std::getenv("HX_JAC_STATS")) {
        unsigned long long z[2];
        CK(cudaStreamSynchronize(s));
        CK(cudaMemcpyFromSymbol(z, g_jac_stats, sizeof(z)));
        std::fprintf(stderr, "[hx jacobi] warp jobs %llu mean sweeps %.2f\n", z[0],
                     z[0] ? double(z[1]) / double(z[0]) : 0.0);
      }
      pm.mark("qr-Bt+jacobi", s);
      // rank selection
      std::vector<SelJob> sj;
      for (size_t a = 0; a < active.size(); ++a) {
        FarBlock& f = fb[active[a]];
        const int exact = (f.dense || (!f.implicit && f.l == f.mu)) ? 1 : 0;
        if (f.implicit)
          sj.push_back(SelJob{f.sig, c->est.p + a, f.l, f.mu, 0, 2});
        else if (explicit_tail && !exact)
          sj.push_back(SelJob{f.sig, c->resid.p + a, f.l, f.mu, 0, 1});
        else
          sj.push_back(SelJob{f.sig, f.fro2, f.l, f.mu, exact, 0});
      }
      c->sel_jobs.upload(sj, s);
      c->rank_d.ensure(size_t(na));
      c->retry_d.ensure(size_t(na));
      select_rank_kernel<<<(na + 127) / 128, 128, 0, s>>>(c->sel_jobs.p, na, cfg->policy,
                                                          cfg->eps, cfg->k_max, over,
                                                          c->rank_d.p, c->retry_d.p, 0);
      CK(cudaGetLastError());
      c->launches++;
      std::vector<int> rk(na), rt(na);
      c->d2h(rk.data(), c->rank_d.p, na * sizeof(int), s);
      c->d2h(rt.data(), c->retry_d.p, na * sizeof(int), s);
      pm.mark("select", s);
      std::vector<int> next;
      for (int a = 0; a < na; ++a) {
        FarBlock& f = fb[active[a]];
        f.rank = rk[a];
        if (rt[a] && f.l < f.mu) next.push_back(active[a]);
        else f.done = 1;
      }
      active.swap(next);
      ++rounds;
    }
    CK(cudaEventRecord(c->ev[3], s));
    for (const FarBlock& f : fb) {
      if (iterative || P->trad) break;
      int& h = c->rank_hint[ilog2(f.mu)];
      h = std::max(h, f.rank);
      if (f.round > 0) c->class_retry[ilog2(f.mu)] = 1;
    }

    hm.mark("recomp-done");
    nvtx.next("hx::output");
    // ---- 4. output factors
    const int nf = int(fb.size());
    c->res_rank.assign(nl, -1);
    c->res_deg.assign(nl, 0);
    c->res_off.assign(nl, 0);
    int64_t pos = 0;
    int64_t max_rank = 0;
    int64_t n_degraded = 0;
    for (const FarBlock& f : fb) {
      c->res_rank[f.leaf] = f.rank;
      c->res_deg[f.leaf] = int8_t(f.degraded ? 1 : 0);
      n_degraded += f.degraded ? 1 : 0;
      c->res_off[f.leaf] = pos;
      pos += int64_t(f.m + f.n) * f.rank;
      max_rank = std::max<int64_t>(max_rank, f.rank);
    }
    c->out_far = pos;
    c->own[BUF_OUT].ensure(size_t(std::max<int64_t>(pos, 1)));
    double* out = c->own[BUF_OUT].p;
    {
      std::vector<int64_t> offs;
      for (const FarBlock& f : fb) offs.push_back(c->res_off[f.leaf]);
      launch_far_outputs(c, fb, offs, out);
    }
    pm.mark("output", s);
    // near leaves: payload stays in BUF_TILE after the far blocks
    c->near_begin = P->near_ws_begin;
    c->near_elems = P->tile_elems - P->near_ws_begin;
    for (int i = 0; i < nl; ++i) {
      const OutLeaf& L = P->leaves[i];
      if (L.kind == 2) c->res_off[i] = c->out_far + (L.ws_off - P->near_ws_begin);
    }
    CK(cudaEventRecord(c->ev[4], s));
    hm.mark("out-issued");
    CK(cudaEventSynchronize(c->ev[4]));
    hm.mark("synced");
    c->trad_release(false);  // finished traditional-mode values are in BUF_OUT now

    if (st) {
      std::memset(st, 0, sizeof(*st));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, c->ev[0], c->ev[4]));
      st->ms_total = ms;
      CK(cudaEventElapsedTime(&ms, c->ev[5], c->ev[1]));
      st->ms_form = ms;
      CK(cudaEventElapsedTime(&ms, c->ev[0], c->ev[5]));
      st->ms_upload = ms;
      CK(cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]));
      st->ms_mat = ms;
      st->dom_kernel_ms = ms;
      CK(cudaEventElapsedTime(&ms, c->ev[2], c->ev[4]));
      st->ms_recompress = ms;
      st->far_leaves = nf;
      st->near_leaves = nl - nf;
      st->degraded_blocks = n_degraded;
      st->sketch_cols = sketch_cols;
      st->max_far_rank = max_rank;
      st->matvec_count = matvecs;
      st->sketch_rounds = rounds;
      st->launches = c->launches;
      st->out_elems = c->out_far + c->near_elems;
      std::vector<double> f2(nl);
      if (nl) c->d2h(f2.data(), c->fro2.p, nl * sizeof(double), s);
      double tot = 0;
      for (double v : f2) tot += v;
      st->fro2_total = tot;
      const int marks[4] = {0, 1, 2, 4};
      for (int k = 0; k < 4; ++k) {
        st->t_marks[k] = -1.0;
        if (g_epoch_set) {
          float t = 0;
          if (cudaEventElapsedTime(&t, g_epoch, c->ev[marks[k]]) == cudaSuccess)
            st->t_marks[k] = t;
          else
            cudaGetLastError();
        }
      }
    }
    return HX_OK;
  });
}

extern "C" int hx_result_layout(hx_ctx* c, int32_t* rank, int8_t* degraded, int64_t* offset) {
  if (!c) return fail(HX_EINVAL, "null ctx");
  const size_t n = c->res_rank.size();
  if (rank) std::copy(c->res_rank.begin(), c->res_rank.end(), rank);
  if (degraded) std::copy(c->res_deg.begin(), c->res_deg.end(), degraded);
  if (offset) std::copy(c->res_off.begin(), c->res_off.end(), offset);
  (void)n;
  return HX_OK;
}

extern "C" int hx_result_download(hx_ctx* c, double* host, int64_t n) {
  return guarded([&]() -> int {
    if (!c || !host) return fail(HX_EINVAL, "null argument");
    if (n < c->out_far + c->near_elems) return fail(HX_EINVAL, "result buffer too small");
    CK(cudaSetDevice(c->device));
    if (c->out_far)
      CK(cudaMemcpyAsync(host, c->own[BUF_OUT].p, size_t(c->out_far) * sizeof(double),
                         cudaMemcpyDeviceToHost, c->s));
    if (c->near_elems)
      CK(cudaMemcpyAsync(host + c->out_far, c->own[BUF_TILE].p + c->near_begin,
                         size_t(c->near_elems) * sizeof(double), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    return HX_OK;
  });
}

extern "C" int hx_debug_gemm(int tile, const void* terms, int64_t n_terms, const void* tiles,
                             int64_t n_tiles, const void* groups, int64_t n_groups,
                             double* const* host_bufs, const int64_t* buf_elems, double* sumsq,
                             int64_t n_sumsq) {
  return guarded([&]() -> int {
    // tile -64: the 64-tile kernel configured for short-K batches (term formation)
    const bool short_k = tile == -64;
    if (short_k) tile = 64;
    if ((tile != 32 && tile != 64) || !terms || !tiles || !groups || !host_bufs || !buf_elems)
      return fail(HX_EINVAL, "bad arguments");
    cudaStream_t s = nullptr;
    hx_ctx tmp;
    tmp.s = s;
    DArr<Term> dt;
    DArr<Tile> dl;
    DArr<Group> dg;
    DArr<double> ds;
    dt.upload(static_cast<const Term*>(terms), size_t(n_terms), s);
    dl.upload(static_cast<const Tile*>(tiles), size_t(n_tiles), s);
    dg.upload(static_cast<const Group*>(groups), size_t(n_groups), s);
    ds.ensure(size_t(std::max<int64_t>(n_sumsq, 1)));
    std::vector<DArr<double>> db(NUM_BUFS);
    BufPtrs bp;
    for (int i = 0; i < NUM_BUFS; ++i) {
      bp.p[i] = nullptr;
      if (host_bufs[i] && buf_elems[i] > 0) {
        db[i].upload(host_bufs[i], size_t(buf_elems[i]), s);
        bp.p[i] = db[i].p;
      }
    }
    launch_gemm(&tmp, tile, dl.p, dg.p, dt.p, int(n_tiles), bp, ds.p, nullptr, short_k);
    CK(cudaDeviceSynchronize());
    for (int i = 0; i < NUM_BUFS; ++i)
      if (bp.p[i])
        CK(cudaMemcpy(host_bufs[i], db[i].p, size_t(buf_elems[i]) * 8, cudaMemcpyDeviceToHost));
    if (sumsq && n_sumsq > 0)
      CK(cudaMemcpy(sumsq, ds.p, size_t(n_sumsq) * 8, cudaMemcpyDeviceToHost));
    for (auto& d : db) d.release();
    dt.release();
    dl.release();
    dg.release();
    ds.release();
    tmp.s = nullptr;
    return HX_OK;
  });
}

extern "C" int hx_debug_qr(int n_jobs, const int32_t* p, const int32_t* q, double* X,
                           double* R) {
  return guarded([&]() -> int {
    if (n_jobs < 0 || (n_jobs && (!p || !q || !X || !R))) return fail(HX_EINVAL, "bad arguments");
    int64_t nx = 0, nr = 0;
    for (int i = 0; i < n_jobs; ++i) {
      if (p[i] < 1 || q[i] < 1 || q[i] > JAC_QMAX || q[i] > p[i])
        return fail(HX_EINVAL, "bad panel shape");
      nx += int64_t(p[i]) * q[i];
      nr += int64_t(q[i]) * q[i];
    }
    hx_ctx tmp;
    tmp.s = nullptr;
    DArr<double> dx, dr;
    dx.upload(X, size_t(nx), nullptr);
    dr.ensure(size_t(std::max<int64_t>(nr, 1)));
    std::vector<QrJob> jobs;
    int64_t ox = 0, orr = 0;
    for (int i = 0; i < n_jobs; ++i) {
      jobs.push_back(QrJob{dx.p + ox, dr.p + orr, p[i], q[i]});
      ox += int64_t(p[i]) * q[i];
      orr += int64_t(q[i]) * q[i];
    }
    run_qr(&tmp, jobs);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(X, dx.p, size_t(nx) * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(R, dr.p, size_t(nr) * 8, cudaMemcpyDeviceToHost));
    dx.release();
    dr.release();
    tmp.qr_jobs.release();
    tmp.ts_jobs.release();
    tmp.tsqr_ws.release();
    return HX_OK;
  });
}

// numpy's default_rng(seed).standard_normal(n) with seed = seed_hi * 2^64 + seed_lo, from
// the host (device < 0) or the device generator (np_random.cuh; parity tests).
extern "C" int hx_np_normals(uint64_t seed_lo, uint64_t seed_hi, int64_t n, double* out,
                             int device) {
  return guarded([&]() -> int {
    if (n < 0 || (n && !out)) return fail(HX_EINVAL, "bad arguments");
    if (device < 0) {
      NpRng g;
      g.seed(seed_lo, seed_hi);
      for (int64_t e = 0; e < n; ++e) out[e] = g.normal();
      return HX_OK;
    }
    CK(cudaSetDevice(device));
    DArr<double> d;
    d.ensure(size_t(std::max<int64_t>(n, 1)));
    np_normals_kernel<<<1, 32>>>(seed_lo, seed_hi, d.p, n);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    if (n) CK(cudaMemcpy(out, d.p, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost));
    d.release();
    return HX_OK;
  });
}

// One block through the matrix-free compressor route of hx_product (tag 0 aca,
// 1 bilanczos, 2 randomized; compressors.py:162-428) on a dense column-major m x n host
// matrix: the per-block stream is default_rng((seed << 24) ^ node).  left (m x rank) and
// right (n x rank) receive the factors (room for min(m, n) columns each); info[0..2] =
// rank, degraded flag, matvec count.
extern "C" int hx_debug_compress(int tag, int policy, double eps, int k_max, int q,
                                 uint64_t seed, int32_t node, int m, int n, const double* A,
                                 double* left, double* right, int32_t* info) {
  hx_ctx* c = nullptr;
  const int rc = guarded([&]() -> int {
    if (tag < 0 || tag > 2 || m < 1 || n < 1 || !A || !left || !right || !info)
      return fail(HX_EINVAL, "bad arguments");
    if (policy == 0 && !(eps > 0.0)) return fail(HX_EINVAL, "eps must be positive");
    if (policy == 1 && k_max < 1) return fail(HX_EINVAL, "k_max must be >= 1");
    const int st = hx_ctx_create(0, &c);
    if (st != HX_OK) return st;
    c->own[BUF_TILE].upload(A, size_t(m) * n, c->s);
    hx_plan P;
    P.leaves.resize(1);
    OutLeaf& L = P.leaves[0];
    std::memset(&L, 0, sizeof(L));
    L.id = node;
    L.kind = 1;
    L.m = m;
    L.n = n;
    std::vector<FarBlock> fb(1);
    fb[0].leaf = 0;
    fb[0].m = m;
    fb[0].n = n;
    fb[0].mu = std::min(m, n);
    fb[0].t_off = 0;
    hx_product_cfg cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.policy = policy;
    cfg.eps = policy == 0 ? eps : 1.0;
    cfg.k_max = k_max;
    cfg.tag = tag;
    cfg.seed = seed;
    cfg.q = q;
    int rounds = 0;
    const int64_t mv = recompress_iterative(c, &P, &cfg, fb, 1, rounds);
    const int r = fb[0].rank;
    c->own[BUF_OUT].ensure(size_t(std::max<int64_t>(int64_t(m + n) * r, 1)));
    launch_far_outputs(c, fb, std::vector<int64_t>{0}, c->own[BUF_OUT].p);
    CK(cudaStreamSynchronize(c->s));
    if (r) {
      CK(cudaMemcpy(left, c->own[BUF_OUT].p, size_t(m) * r * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(right, c->own[BUF_OUT].p + int64_t(m) * r, size_t(n) * r * 8,
                    cudaMemcpyDeviceToHost));
    }
    info[0] = r;
    info[1] = fb[0].degraded;
    info[2] = int32_t(mv);
    return HX_OK;
  });
  if (c) hx_ctx_free(c);
  return rc;
}

// H-matrix times a block of s vectors, Y = M X or M^T X (hmat_vec / _node_matmat,
// hmatrix.py:138-202), for the operand in slot `which` of the context.  The same grouped
// GEMM as the product: cores W_l = V_l^T X[sigma_l] stacked, then row bands of Y summing
// U_l W_l and D_l X[sigma_l] over the leaves covering each band.
extern "C" int hx_hmatvec(hx_ctx* c, const hx_tree* tree, const hx_operand* op, int which,
                          int transpose, const double* X, double* Y, int s) {
  return guarded([&]() -> int {
    if (!c || !tree || !op || !X || !Y || s < 1 || which < 0 || which > 1)
      return fail(HX_EINVAL, "bad arguments");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->s;
    const int64_t n = tree->c_hi[0] - tree->c_lo[0];
    auto lo = [&](int cl) { return tree->c_lo[cl]; };
    auto sz = [&](int cl) { return tree->c_hi[cl] - tree->c_lo[cl]; };
    // input rows / output rows of a leaf
    auto in_cl = [&](int b) { return transpose ? tree->tau[b] : tree->sigma[b]; };
    auto out_cl = [&](int b) { return transpose ? tree->sigma[b] : tree->tau[b]; };
    std::vector<int> lr, dn;
    std::vector<int64_t> off;
    int64_t srows = 0;
    for (int b = 0; b < tree->n_nodes; ++b) {
      if (tree->kind[b] == 0) continue;
      if (op->payload[b] == 1) {
        if (op->rank[b] == 0) continue;
        lr.push_back(b);
        off.push_back(srows);
        srows += op->rank[b];
      } else {
        dn.push_back(b);
      }
    }
    std::vector<Term> terms;
    std::vector<Group> groups;
    std::vector<Tile> tiles;
    const int T = 64;
    auto tiles_over = [&](uint8_t out_buf, int64_t R, int64_t C, int32_t gbase) {
      for (int64_t i = 0, band = 0; i < R; i += T, ++band)
        for (int64_t j = 0; j < C; j += T) {
          Tile t;
          std::memset(&t, 0, sizeof(t));
          t.out_off = i + j * R;
          t.out_ld = int32_t(R);
          t.row0 = int32_t(i);
          t.col0 = int32_t(j);
          t.rows = int16_t(std::min<int64_t>(T, R - i));
          t.cols = int16_t(std::min<int64_t>(T, C - j));
          t.g_begin = gbase + int32_t(band);
          t.g_end = t.g_begin + 1;
          t.aux = -1;
          t.out_buf = out_buf;
          t.mode = MODE_STORE;
          tiles.push_back(t);
        }
    };
    // cores: S rows [off_l, off_l + k_l) = (V_l or U_l)^T X[in rows]
    const int64_t nbs = (srows + T - 1) / T;
    {
      std::vector<std::vector<Term>> bands(static_cast<size_t>(nbs));
      for (size_t q = 0; q < lr.size(); ++q) {
        const int b = lr[q];
        const int k = op->rank[b];
        const int ic = in_cl(b);
        const int64_t f = transpose ? op->u_off[b] : op->v_off[b];
        const Term tm = mk(uint8_t(which), f, int32_t(sz(ic)), 1, BUF_GATHER, lo(ic), int32_t(n),
                           1, int32_t(sz(ic)), k, s);
        Term t2 = tm;
        t2.r_lo = int32_t(off[q]);
        for (int64_t bb = off[q] / T; bb <= (off[q] + k - 1) / T; ++bb) bands[size_t(bb)].push_back(t2);
      }
      for (auto& v : bands) {
        groups.push_back(Group{int32_t(terms.size()), int32_t(terms.size() + v.size())});
        terms.insert(terms.end(), v.begin(), v.end());
      }
      tiles_over(BUF_CORE, srows, s, 0);
    }
    const size_t core_tiles = tiles.size();
    // Y bands
    const int64_t nb = (n + T - 1) / T;
    const int32_t gy = int32_t(groups.size());
    {
      std::vector<std::vector<Term>> bands(static_cast<size_t>(nb));
      for (size_t q = 0; q < lr.size(); ++q) {
        const int b = lr[q];
        const int k = op->rank[b];
        const int oc = out_cl(b);
        const int64_t f = transpose ? op->v_off[b] : op->u_off[b];
        const Term tm = mk(uint8_t(which), f, int32_t(sz(oc)), 0, BUF_CORE, off[q],
                           int32_t(srows), 1, k, int32_t(sz(oc)), s);
        Term t2 = tm;
        t2.r_lo = int32_t(lo(oc));
        for (int64_t bb = lo(oc) / T; bb <= (lo(oc) + sz(oc) - 1) / T; ++bb)
          bands[size_t(bb)].push_back(t2);
      }
      for (int b : dn) {
        const int oc = out_cl(b), ic = in_cl(b);
        // D (tau x sigma, ld |tau|): forward P = D (i-contig), transpose P = D^T (k-contig)
        Term t2 = mk(uint8_t(which), op->d_off[b], int32_t(sz(tree->tau[b])),
                     uint8_t(transpose ? 1 : 0), BUF_GATHER, lo(ic), int32_t(n), 1,
                     int32_t(sz(ic)), int32_t(sz(oc)), s);
        t2.r_lo = int32_t(lo(oc));
        for (int64_t bb = lo(oc) / T; bb <= (lo(oc) + sz(oc) - 1) / T; ++bb)
          bands[size_t(bb)].push_back(t2);
      }
      for (auto& v : bands) {
        groups.push_back(Group{int32_t(terms.size()), int32_t(terms.size() + v.size())});
        terms.insert(terms.end(), v.begin(), v.end());
      }
      tiles_over(BUF_TERM, n, s, gy);
    }
    DArr<double> dx, dy, ds;
    DArr<Term> dt;
    DArr<Tile> dl;
    DArr<Group> dg;
    dx.upload(X, size_t(n) * s, st);
    dy.ensure(size_t(n) * s);
    ds.ensure(size_t(std::max<int64_t>(srows, 1)) * s);
    dt.upload(terms, st);
    dl.upload(tiles, st);
    dg.upload(groups, st);
    BufPtrs bp = c->ptrs();
    bp.p[BUF_GATHER] = dx.p;
    bp.p[BUF_CORE] = ds.p;
    bp.p[BUF_TERM] = dy.p;
    launch_gemm(c, 64, dl.p, dg.p, dt.p, int(core_tiles), bp, nullptr);
    launch_gemm(c, 64, dl.p + core_tiles, dg.p, dt.p, int(tiles.size() - core_tiles), bp,
                nullptr);
    CK(cudaMemcpyAsync(Y, dy.p, size_t(n) * s * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    dx.release();
    dy.release();
    ds.release();
    dt.release();
    dl.release();
    dg.release();
    return HX_OK;
  });
}

static size_t ctx_held(const hx_ctx* c) {
  size_t held = 0;
  for (int i = 0; i < NUM_BUFS; ++i)
    if (i != BUF_A && i != BUF_B && i != BUF_WORK) held += c->own[i].cap * sizeof(double);
  for (const auto& w : c->work) held += w.cap * sizeof(double);
  return held;
}

extern "C" int hx_ctx_mem_info(hx_ctx* c, int64_t* free_bytes, int64_t* total_bytes) {
  return guarded([&]() -> int {
    if (!c) return fail(HX_EINVAL, "null ctx");
    CK(cudaSetDevice(c->device));
    size_t f = 0, t = 0;
    CK(cudaMemGetInfo(&f, &t));
    // memory this context already holds for reuse counts as available
    if (free_bytes) *free_bytes = int64_t(f + ctx_held(c));
    if (total_bytes) *total_bytes = int64_t(t);
    return HX_OK;
  });
}

extern "C" int64_t hx_ctx_held_bytes(hx_ctx* c) { return c ? int64_t(ctx_held(c)) : 0; }

extern "C" int hx_ctx_synchronize(hx_ctx* c) {
  return guarded([&]() -> int {
    if (!c) return fail(HX_EINVAL, "null ctx");
    CK(cudaStreamSynchronize(c->s));
    return HX_OK;
  });
}

extern "C" void hx_ctx_free(hx_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->s);
  for (auto& b : c->own) {
    if (&b == &c->own[BUF_WORK]) continue;  // points into work[]
    b.release();
  }
  for (auto& w : c->work) w.release();
  c->trad_release(true);
  for (double* p : c->pools) cudaFree(p);
  for (int i = 0; i < 3; ++i) {
    c->terms[i].release();
    c->tiles[i].release();
    c->groups[i].release();
  }
  c->sumsq.release();
  c->fro2.release();
  c->seg_b.release();
  c->seg_e.release();
  c->gcols.release();
  c->rterms.release();
  c->rtiles.release();
  c->rgroups.release();
  c->qr_jobs.release();
  c->jac_jobs.release();
  c->sel_jobs.release();
  c->small_jobs.release();
  c->rank_d.release();
  c->retry_d.release();
  for (auto& e : c->ev) cudaEventDestroy(e);
  cudaEventDestroy(c->up_ev);
  cudaStreamDestroy(c->s);
  cudaStreamDestroy(c->s2);
  cudaStreamDestroy(c->s_hi);
  cudaStreamDestroy(c->s3);
  if (c->stage) hx::pinned_free(c->stage, c->stage_bytes);
  delete c;
}

#include "assemble.cuh"

// ---- page-locked host memory for the Python layer (result blocks, operand pools)
extern "C" void* hx_host_alloc(int64_t bytes) {
  try {
    return hx::pinned_alloc(size_t(std::max<int64_t>(bytes, 1)));
  } catch (...) {
    return nullptr;
  }
}

extern "C" void hx_host_free(void* p, int64_t bytes) {
  hx::pinned_free(p, size_t(std::max<int64_t>(bytes, 1)));
}

extern "C" int hx_host_register(void* p, int64_t bytes) {
  if (!p || bytes <= 0) return fail(HX_EINVAL, "bad host range");
  const cudaError_t e = cudaHostRegister(p, size_t(bytes), cudaHostRegisterPortable);
  if (e == cudaSuccess) return HX_OK;
  cudaGetLastError();
  if (e == cudaErrorHostMemoryAlreadyRegistered) return HX_OK;
  return fail(HX_ECUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e));
}

extern "C" int hx_host_unregister(void* p) {
  if (!p) return HX_OK;
  if (cudaHostUnregister(p) != cudaSuccess) cudaGetLastError();
  return HX_OK;
}

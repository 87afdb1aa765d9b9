// HMX1 operator files: the on-disk interchange of assembled operands.
//
// Byte format of the reference (pkg/src/hmat/hmatrix.py:9-24), little endian:
//   "HMX1", u32 version (1), u64 n, 32-byte sha256 of the block-tree dump, u64 count,
//   then per leaf in ascending node id (save_hmatrix, hmatrix.py:338-361):
//   u64 node_id, u8 kind (0 dense, 1 low rank), u8 degraded,
//   dense: u32 m, u32 n, m*n f64 row-major; low rank: u32 m, n, k, m*k f64 (left),
//   n*k f64 (right), both row-major.
//
// The reference writes and reads leaf by leaf through Python objects.  Here the file maps
// straight onto the packed column-major operand pool the GPU consumes (hx_operand_layout):
// the writer transposes windows of records in parallel and streams them out; the reader
// scans the record headers once (hx_hmx1_scan: payload kinds, ranks, degraded flags,
// payload positions), the caller lays the pool out, and hx_hmx1_read fills it with
// parallel positioned reads.  Header checks and their messages follow load_hmatrix
// (hmatrix.py:364-388).
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hx.h"
#include "hx_internal.h"

namespace {

constexpr size_t HEADER = 4 + 4 + 8 + 32 + 8;
constexpr size_t WINDOW = size_t(256) << 20;  // bytes of records transposed per write

struct Leaf {
  int32_t id;
  int8_t kind;  // 0 dense, 1 low rank (file kinds)
  int64_t m, n, k;
  int64_t bytes;  // record size
};

int64_t dim(const hx_tree* t, int32_t c) { return t->c_hi[c] - t->c_lo[c]; }

template <class T>
void put(char*& p, T v) {
  std::memcpy(p, &v, sizeof(T));
  p += sizeof(T);
}

// row-major m x k from column-major (ld m)
void to_rows(const double* col, int64_t m, int64_t k, double* out) {
  constexpr int64_t B = 32;
  for (int64_t i0 = 0; i0 < m; i0 += B)
    for (int64_t j0 = 0; j0 < k; j0 += B)
      for (int64_t i = i0; i < std::min(m, i0 + B); ++i)
        for (int64_t j = j0; j < std::min(k, j0 + B); ++j) out[i * k + j] = col[i + j * m];
}

void to_cols(const double* row, int64_t m, int64_t k, double* out) {
  constexpr int64_t B = 32;
  for (int64_t j0 = 0; j0 < k; j0 += B)
    for (int64_t i0 = 0; i0 < m; i0 += B)
      for (int64_t j = j0; j < std::min(k, j0 + B); ++j)
        for (int64_t i = i0; i < std::min(m, i0 + B); ++i) out[i + j * m] = row[i * k + j];
}

bool pread_all(int fd, void* dst, size_t bytes, int64_t pos) {
  char* p = static_cast<char*>(dst);
  while (bytes) {
    const ssize_t r = ::pread(fd, p, bytes, off_t(pos));
    if (r <= 0) return false;
    p += r;
    pos += r;
    bytes -= size_t(r);
  }
  return true;
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

}  // namespace

extern "C" int hx_hmx1_write(const char* path, const hx_tree* tree, int64_t n,
                             const uint8_t* fingerprint, const hx_operand* op,
                             const int8_t* degraded, const double* pool) {
  return hx::guarded([&]() -> int {
    if (!path || !tree || !fingerprint || !op || !pool) return hx::fail(HX_EINVAL, "null argument");
    std::vector<Leaf> leaves;
    for (int32_t b = 0; b < tree->n_nodes; ++b) {
      const int8_t pl = op->payload[b];
      if (pl == 0) continue;
      Leaf L;
      L.id = b;
      L.m = dim(tree, tree->tau[b]);
      L.n = dim(tree, tree->sigma[b]);
      if (pl == 1) {
        L.kind = 1;
        L.k = op->rank[b];
        L.bytes = 8 + 2 + 12 + 8 * L.k * (L.m + L.n);
      } else {
        L.kind = 0;
        L.k = 0;
        L.bytes = 8 + 2 + 8 + 8 * L.m * L.n;
      }
      leaves.push_back(L);
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) return hx::fail(HX_EINVAL, std::string("cannot open ") + path + " for writing");
    struct Closer {
      FILE* f;
      ~Closer() {
        if (f) std::fclose(f);
      }
    } closer{f};
    char head[HEADER];
    char* p = head;
    std::memcpy(p, "HMX1", 4);
    p += 4;
    put<uint32_t>(p, 1u);
    put<uint64_t>(p, uint64_t(n));
    std::memcpy(p, fingerprint, 32);
    p += 32;
    put<uint64_t>(p, uint64_t(leaves.size()));
    if (std::fwrite(head, 1, HEADER, f) != HEADER) return hx::fail(HX_EINVAL, "write failed");
    int64_t biggest = 0;
    for (const Leaf& L : leaves) biggest = std::max(biggest, L.bytes);
    std::vector<char> buf(std::max<size_t>(WINDOW, size_t(biggest)));
    std::vector<int64_t> at;
    for (size_t a = 0; a < leaves.size();) {
      size_t e = a;
      int64_t used = 0;
      at.clear();
      while (e < leaves.size() && (e == a || used + leaves[e].bytes <= int64_t(buf.size()))) {
        at.push_back(used);
        used += leaves[e].bytes;
        ++e;
      }
#pragma omp parallel for schedule(dynamic, 64)
      for (int64_t i = 0; i < int64_t(e - a); ++i) {
        const Leaf& L = leaves[a + size_t(i)];
        char* q = buf.data() + at[size_t(i)];
        put<uint64_t>(q, uint64_t(L.id));
        put<uint8_t>(q, uint8_t(L.kind));
        put<uint8_t>(q, uint8_t(degraded && degraded[L.id] ? 1 : 0));
        put<uint32_t>(q, uint32_t(L.m));
        put<uint32_t>(q, uint32_t(L.n));
        if (L.kind == 1) {
          put<uint32_t>(q, uint32_t(L.k));
          std::vector<double> tmp(size_t(std::max(L.m, L.n) * L.k));  // records are unaligned
          to_rows(pool + op->u_off[L.id], L.m, L.k, tmp.data());
          std::memcpy(q, tmp.data(), size_t(8 * L.m * L.k));
          to_rows(pool + op->v_off[L.id], L.n, L.k, tmp.data());
          std::memcpy(q + 8 * L.m * L.k, tmp.data(), size_t(8 * L.n * L.k));
        } else {
          std::vector<double> tmp(size_t(L.m * L.n));
          to_rows(pool + op->d_off[L.id], L.m, L.n, tmp.data());
          std::memcpy(q, tmp.data(), size_t(8 * L.m * L.n));
        }
      }
      if (std::fwrite(buf.data(), 1, size_t(used), f) != size_t(used))
        return hx::fail(HX_EINVAL, "write failed");
      a = e;
    }
    if (std::fclose(f) != 0) {
      closer.f = nullptr;
      return hx::fail(HX_EINVAL, "write failed");
    }
    closer.f = nullptr;
    return HX_OK;
  });
}

extern "C" int hx_hmx1_scan(const char* path, const hx_tree* tree, int64_t n,
                            const uint8_t* fingerprint, int8_t* payload, int32_t* rank,
                            int8_t* degraded, int64_t* pos) {
  return hx::guarded([&]() -> int {
    if (!path || !tree || !fingerprint || !payload || !rank || !degraded || !pos)
      return hx::fail(HX_EINVAL, "null argument");
    Fd fd;
    fd.fd = ::open(path, O_RDONLY);
    if (fd.fd < 0) return hx::fail(HX_EINVAL, std::string("cannot open ") + path);
    char head[HEADER];
    if (!pread_all(fd.fd, head, 4, 0) || std::memcmp(head, "HMX1", 4) != 0)
      return hx::fail(HX_EINVAL, "not an H-matrix file");
    if (!pread_all(fd.fd, head + 4, HEADER - 4, 4)) return hx::fail(HX_EINVAL, "truncated H-matrix file");
    uint32_t version;
    uint64_t fn, count;
    std::memcpy(&version, head + 4, 4);
    std::memcpy(&fn, head + 8, 8);
    std::memcpy(&count, head + 48, 8);
    if (version != 1) return hx::fail(HX_EINVAL, "unsupported version " + std::to_string(version));
    if (int64_t(fn) != n)
      return hx::fail(HX_EINVAL, "dimension mismatch: file " + std::to_string(fn) + ", tree " +
                                     std::to_string(n));
    if (std::memcmp(head + 16, fingerprint, 32) != 0)
      return hx::fail(HX_EINVAL, "block tree does not match the stored operator");
    const int32_t nn = tree->n_nodes;
    std::fill(payload, payload + nn, int8_t(0));
    std::fill(rank, rank + nn, 0);
    std::fill(degraded, degraded + nn, int8_t(0));
    std::fill(pos, pos + nn, int64_t(-1));
    int64_t at = int64_t(HEADER);
    for (uint64_t r = 0; r < count; ++r) {
      char rec[22];
      if (!pread_all(fd.fd, rec, 10, at)) return hx::fail(HX_EINVAL, "truncated H-matrix file");
      uint64_t id;
      std::memcpy(&id, rec, 8);
      const uint8_t kind = uint8_t(rec[8]), flag = uint8_t(rec[9]);
      const int hdr = kind == 1 ? 12 : 8;
      if (!pread_all(fd.fd, rec + 10, size_t(hdr), at + 10))
        return hx::fail(HX_EINVAL, "truncated H-matrix file");
      uint32_t m, nc, k = 0;
      std::memcpy(&m, rec + 10, 4);
      std::memcpy(&nc, rec + 14, 4);
      if (kind == 1) std::memcpy(&k, rec + 18, 4);
      if (id >= uint64_t(nn) || tree->kind[id] == 0 || kind > 1)
        return hx::fail(HX_EINVAL, "record " + std::to_string(r) + ": node " +
                                       std::to_string(id) + " is not a leaf of the tree");
      if (int64_t(m) != dim(tree, tree->tau[id]) || int64_t(nc) != dim(tree, tree->sigma[id]))
        return hx::fail(HX_EINVAL, "record for node " + std::to_string(id) +
                                       " does not match the block shape");
      payload[id] = kind == 1 ? 1 : 2;
      rank[id] = int32_t(k);
      degraded[id] = flag ? 1 : 0;
      pos[id] = at + 10 + hdr;
      at += 10 + hdr + 8 * (kind == 1 ? int64_t(k) * (int64_t(m) + nc) : int64_t(m) * nc);
    }
    for (int32_t b = 0; b < nn; ++b)
      if (tree->kind[b] != 0 && payload[b] == 0)
        return hx::fail(HX_EINVAL, "no payload for leaf " + std::to_string(b));
    return HX_OK;
  });
}

extern "C" int hx_hmx1_read(const char* path, const hx_tree* tree, const hx_operand* op,
                            const int64_t* pos, double* pool) {
  return hx::guarded([&]() -> int {
    if (!path || !tree || !op || !pos || !pool) return hx::fail(HX_EINVAL, "null argument");
    Fd fd;
    fd.fd = ::open(path, O_RDONLY);
    if (fd.fd < 0) return hx::fail(HX_EINVAL, std::string("cannot open ") + path);
    std::vector<int32_t> ids;
    for (int32_t b = 0; b < tree->n_nodes; ++b)
      if (op->payload[b] != 0) ids.push_back(b);
    int bad = 0;
#pragma omp parallel
    {
      std::vector<double> tmp;
#pragma omp for schedule(dynamic, 64) reduction(+ : bad)
      for (int64_t i = 0; i < int64_t(ids.size()); ++i) {
        const int32_t b = ids[size_t(i)];
        const int64_t m = dim(tree, tree->tau[b]), n = dim(tree, tree->sigma[b]);
        if (op->payload[b] == 1) {
          const int64_t k = op->rank[b];
          tmp.resize(size_t(std::max<int64_t>(1, k * (m + n))));
          if (!pread_all(fd.fd, tmp.data(), size_t(8 * k * (m + n)), pos[b])) {
            ++bad;
            continue;
          }
          to_cols(tmp.data(), m, k, pool + op->u_off[b]);
          to_cols(tmp.data() + m * k, n, k, pool + op->v_off[b]);
        } else {
          tmp.resize(size_t(std::max<int64_t>(1, m * n)));
          if (!pread_all(fd.fd, tmp.data(), size_t(8 * m * n), pos[b])) {
            ++bad;
            continue;
          }
          to_cols(tmp.data(), m, n, pool + op->d_off[b]);
        }
      }
    }
    if (bad) return hx::fail(HX_EINVAL, "truncated H-matrix file");
    return HX_OK;
  });
}

// Internal device/host descriptor types shared by the plan builder and the CUDA kernels.
//
// The whole product is expressed as batches of "tiles": one tile is one CTA's output
// region (at most TM x TN doubles) that receives a sum of products P_i * Q_i.  A product
// ("term") names its two operands by (buffer id, element offset, leading dimension,
// contiguity) and carries the coordinate origin (r_lo, c_lo) of the block it was created
// on, so that the same term serves every tile of every output block below its creation
// block: the slice a tile needs starts at (tile.row0 - r_lo, tile.col0 - c_lo).
//
//   P (rows x k):  a_kc == 0 -> P(i, kk) = buf[a_off + i + kk * a_ld]   (column-major factor)
//                  a_kc == 1 -> P(i, kk) = buf[a_off + kk + i * a_ld]   (transposed factor)
//   Q (k x cols):  b_kc == 0 -> Q(kk, j) = buf[b_off + j + kk * b_ld]   (factor used as F^T)
//                  b_kc == 1 -> Q(kk, j) = buf[b_off + kk + j * b_ld]   (column-major matrix)
//                  b_kc == 2 -> Q(kk, j) = G(b_off + kk, j), G the tile's column-gathered
//                               virtual matrix (ColRec, MODE_GCOL tiles)
//
// A term only covers rows [r_lo, r_lo + rows) and columns [c_lo, c_lo + cols) of the
// tile coordinate system; the kernel zero-fills outside, so a term created on a
// sub-block of an output block (pending-pair expansion) contributes to its part of a
// tile only.
#pragma once
#include <cstdint>

namespace hx {

enum Buf : uint8_t {
  BUF_A = 0,       // operand A pool (far U/V factors, dense leaves)
  BUF_B = 1,       // operand B pool (aliases A when A is B)
  BUF_TERM = 2,    // computed term factors (V_B core^T, U_A core, X U_B, X^T V_A)
  BUF_CORE = 3,    // k x k cores V_A^T U_B and leaf cores inside X
  BUF_TILE = 4,    // materialized output blocks (column-major m x n per leaf)
  BUF_OMEGA = 5,   // Gaussian test matrix for the sketch
  BUF_WORK = 6,    // recompression workspace (Y/Q, Bt/Q2, small matrices)
  BUF_OUT = 7,     // output factors (left m x r, right n x r per far leaf)
  BUF_GATHER = 8,  // scratch: transposed dense blocks of mixed pairs; X of hx_hmatvec
  BUF_EYE = 9,     // identity matrix (the plain factor of H-block x dense terms)
  NUM_BUFS = 10
};

// Contiguous copy of n doubles from (src_buf, src_off) to BUF_GATHER + dst_off.
struct CopyRec {
  int64_t src_off, dst_off, n;
  int32_t src_buf;
  int32_t pad;
};

// Leading dimension of the identity operand (BUF_EYE): the fixed factor of H-block x dense
// terms, whose rank is a leaf cluster size.
constexpr int EYE_LD = 1024;

// Transposed copy of a dense block (rows x cols, column-major, in BUF_A at src_off) into
// BUF_GATHER at dst_off (cols x rows): the thin matrix of dense x H-block terms.
struct TransRec {
  int64_t src_off, dst_off;
  int32_t rows, cols;
};

// One thin factor of an X-group, seen as columns [col, col + k) of the group's virtual
// matrix G: column col + c is bufs[buf] + src_off + c * ld (ld = |rho| rows).  Tiles in
// MODE_GCOL read G through these records instead of a gathered copy (Term b_kc == 2).
struct ColRec {
  int64_t src_off;
  int32_t col, k, ld, buf;
};
static_assert(sizeof(ColRec) == 24, "ColRec layout");

enum TileMode : uint8_t {
  MODE_STORE = 0,       // out  = sum
  MODE_ADD = 1,         // out += sum
  MODE_STORE_SUMSQ = 2,  // out  = sum, and sumsq[aux] = sum of squares of the tile
  MODE_RESID_SUMSQ = 3,  // out unchanged, sumsq[aux] = sum of squares of (out - sum)
  MODE_GCOL = 4          // out = sum; aux = first ColRec of the tile's columns (b_kc == 2)
};

struct Term {
  int64_t a_off, b_off;
  int32_t a_ld, b_ld;
  int32_t k;
  int32_t r_lo, c_lo;
  int32_t rows, cols;
  uint8_t a_buf, b_buf, a_kc, b_kc;
};
static_assert(sizeof(Term) == 48, "Term layout");

struct Group {
  int32_t t_begin, t_end;  // contiguous range of terms
};

struct Tile {
  int64_t out_off;
  int32_t out_ld;
  int32_t row0, col0;      // coordinates used to slice every term of the tile
  int16_t rows, cols;      // extent (<= TM, TN)
  int32_t g_begin, g_end;  // range of groups
  int32_t aux;             // sum-of-squares slot (MODE_STORE_SUMSQ)
  uint8_t out_buf, mode;
  uint8_t pad[2];
};
static_assert(sizeof(Tile) == 40, "Tile layout");

}  // namespace hx

// numpy's Generator stream, bit for bit, on the host and on the device.
//
// The reference seeds one stream per far block, np.random.default_rng(_block_seed(kind,
// node.id)) with _block_seed = (seed << 24) ^ node.id (multiply.py:61-63), and draws the
// Lanczos start vector / restart probes (compressors.py:303, :318) and the randomized
// probes (:389, :424) with standard_normal.  Reproducing that stream makes the GPU's
// bilanczos / randomized runs follow the reference's own random directions:
//   SeedSequence(seed)  32-bit hashmix entropy pool of 4 words, generate_state(4, uint64)
//   PCG64               128-bit LCG (multiplier 0x2360ED051FC65DA44385DF649FCCF645),
//                       XSL-RR 128 -> 64 output, seeded with (state, increment) words
//   standard_normal     256-layer ziggurat on one 64-bit draw (8 bits layer, 1 sign,
//                       52 magnitude), with the exponential tail and wedge rejections
// The ziggurat tables are numpy's own (zig_tables.inc, generated at build time by
// tools/gen_ziggurat.py); tests/np_random_ref.py is the Python restatement that pins both.
#pragma once
#include <cmath>
#include <cstdint>

#include "zig_tables.inc"

namespace hx {

static const uint64_t hZigKi[256] = {HX_ZIG_KI};
static const double hZigWi[256] = {HX_ZIG_WI};
static const double hZigFi[256] = {HX_ZIG_FI};
#ifdef __CUDACC__
__device__ const uint64_t dZigKi[256] = {HX_ZIG_KI};
__device__ const double dZigWi[256] = {HX_ZIG_WI};
__device__ const double dZigFi[256] = {HX_ZIG_FI};
#define HX_HD __host__ __device__
#else
#define HX_HD
#endif

typedef unsigned __int128 u128;

struct NpRng {
  u128 state, inc;

  // seed = hi * 2^64 + lo: a non-negative Python int of up to 128 bits
  HX_HD void seed(uint64_t lo, uint64_t hi) {
    const uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
    const uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
    const uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
    uint32_t ent[4];
    int n_ent = 0;
    {  // entropy words: little-endian 32-bit chunks, [0] for zero
      uint32_t w[4] = {uint32_t(lo), uint32_t(lo >> 32), uint32_t(hi), uint32_t(hi >> 32)};
      for (int i = 0; i < 4; ++i)
        if (w[i]) n_ent = i + 1;
      if (n_ent == 0) n_ent = 1;
      for (int i = 0; i < 4; ++i) ent[i] = w[i];
    }
    uint32_t hc = kInitA;
    auto hashmix = [&](uint32_t v) {
      v ^= hc;
      hc *= kMultA;
      v *= hc;
      return v ^ (v >> 16);
    };
    auto mix = [&](uint32_t x, uint32_t y) {
      uint32_t r = kMixL * x - kMixR * y;
      return r ^ (r >> 16);
    };
    uint32_t pool[4];
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u);
    for (int s = 0; s < 4; ++s)
      for (int d = 0; d < 4; ++d)
        if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
    // (entropy beyond the 4-word pool cannot occur for <= 128-bit seeds)
    uint32_t hb = kInitB;
    uint64_t v[4];
    for (int i = 0; i < 4; ++i) {
      uint32_t w2[2];
      for (int h = 0; h < 2; ++h) {
        uint32_t x = pool[(2 * i + h) & 3] ^ hb;
        hb *= kMultB;
        x *= hb;
        w2[h] = x ^ (x >> 16);
      }
      v[i] = uint64_t(w2[0]) | (uint64_t(w2[1]) << 32);
    }
    const u128 init = (u128(v[0]) << 64) | v[1];
    const u128 seq = (u128(v[2]) << 64) | v[3];
    inc = (seq << 1) | 1u;
    state = 0;
    step();
    state += init;
    step();
  }
  HX_HD void step() {
    const u128 mult = (u128(0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;
    state = state * mult + inc;
  }
  HX_HD uint64_t next64() {
    step();
    const uint64_t x = uint64_t(state >> 64) ^ uint64_t(state);
    const unsigned rot = unsigned(state >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  HX_HD double next_double() { return double(next64() >> 11) * (1.0 / 9007199254740992.0); }

  HX_HD double normal() {
#ifdef __CUDA_ARCH__
    const uint64_t* ki = dZigKi;
    const double* wi = dZigWi;
    const double* fi = dZigFi;
#else
    const uint64_t* ki = hZigKi;
    const double* wi = hZigWi;
    const double* fi = hZigFi;
#endif
    const double r_tail = 3.6541528853610087963519472518;
    const double inv_r = 0.27366123732975827203338247596;
    for (;;) {
      uint64_t r = next64();
      const int idx = int(r & 0xff);
      r >>= 8;
      const uint64_t sign = r & 1;
      const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
      double x = double(rabs) * wi[idx];
      if (sign) x = -x;
      if (rabs < ki[idx]) return x;
      if (idx == 0) {
        for (;;) {
          const double xx = -inv_r * log1p(-next_double());
          const double yy = -log1p(-next_double());
          if (yy + yy > xx * xx) return ((rabs >> 8) & 1) ? -(r_tail + xx) : r_tail + xx;
        }
      } else if ((fi[idx - 1] - fi[idx]) * next_double() + fi[idx] < exp(-0.5 * x * x)) {
        return x;
      }
    }
  }
};

// The reference's per-block seed (multiply.py:61-63): (seed << 24) ^ node_id as a
// 128-bit value (lo, hi).
HX_HD inline void block_seed(uint64_t seed, int64_t node_id, uint64_t& lo, uint64_t& hi) {
  lo = (seed << 24) ^ uint64_t(node_id);
  hi = seed >> 40;
}

}  // namespace hx

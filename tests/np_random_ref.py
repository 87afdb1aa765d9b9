"""Pure-Python restatement of numpy's ``default_rng(seed).standard_normal`` stream (test
infrastructure: it pins the device generator ``csrc/np_random.cuh`` and the build-time table
extraction ``tools/gen_ziggurat.py``).

numpy 2.x: ``SeedSequence`` (32-bit hashmix pool of 4 words, ``generate_state`` of 4
uint64), ``PCG64`` (128-bit LCG, XSL-RR output), ``Generator.standard_normal``
(256-layer ziggurat on 64-bit draws).  The reference seeds one such stream per far block
(``multiply.py:61-63``) for its Lanczos start vector and randomized probes
(``compressors.py:303, :389, :424``).
"""

import math

import numpy as np

M32 = 0xFFFFFFFF
M64 = (1 << 64) - 1
M128 = (1 << 128) - 1
INIT_A, MULT_A = 0x43B0D7E5, 0x931E8875
INIT_B, MULT_B = 0x8B51F9DD, 0x58F38DED
MIX_L, MIX_R = 0xCA01F9DD, 0x4973F715
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
ZIG_R = 3.6541528853610087963519472518
ZIG_INV_R = 0.27366123732975827203338247596


def seed_words(seed):
    """The entropy of a non-negative int as little-endian 32-bit words."""
    if seed == 0:
        return [0]
    out = []
    while seed > 0:
        out.append(seed & M32)
        seed >>= 32
    return out


def seedseq_state(seed):
    ent = seed_words(int(seed))
    hc = [INIT_A]

    def hashmix(v):
        v ^= hc[0]
        hc[0] = (hc[0] * MULT_A) & M32
        v = (v * hc[0]) & M32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (MIX_L * x - MIX_R * y) & M32
        return r ^ (r >> 16)

    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(4)]
    for s in range(4):
        for d in range(4):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(4, len(ent)):
        for d in range(4):
            pool[d] = mix(pool[d], hashmix(ent[s]))
    h, words = INIT_B, []
    for i in range(8):
        v = pool[i % 4] ^ h
        h = (h * MULT_B) & M32
        v = (v * h) & M32
        words.append(v ^ (v >> 16))
    return [words[2 * i] | (words[2 * i + 1] << 32) for i in range(4)]


class PCG64:
    def __init__(self, seed):
        v = seedseq_state(seed)
        init, seq = (v[0] << 64) | v[1], (v[2] << 64) | v[3]
        self.inc = ((seq << 1) | 1) & M128
        self.state = 0
        self._step()
        self.state = (self.state + init) & M128
        self._step()

    def _step(self):
        self.state = (self.state * PCG_MULT + self.inc) & M128

    def next64(self):
        self._step()
        s = self.state
        x = ((s >> 64) ^ s) & M64
        rot = s >> 122
        return ((x >> rot) | (x << ((64 - rot) & 63))) & M64

    def next_double(self):
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)


def normals(seed, n, ki, wi, fi):
    g = PCG64(seed)
    out = np.empty(n)
    for t in range(n):
        while True:
            r = g.next64()
            idx = r & 0xFF
            r >>= 8
            sign = r & 1
            rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
            x = rabs * float(wi[idx])
            if sign:
                x = -x
            if rabs < int(ki[idx]):
                break
            if idx == 0:
                while True:
                    xx = -ZIG_INV_R * math.log1p(-g.next_double())
                    yy = -math.log1p(-g.next_double())
                    if yy + yy > xx * xx:
                        x = -(ZIG_R + xx) if (rabs >> 8) & 1 else ZIG_R + xx
                        break
                break
            if (float(fi[idx - 1]) - float(fi[idx])) * g.next_double() + float(fi[idx]) < \
                    math.exp(-0.5 * x * x):
                break
        out[t] = x
    return out

"""numpy's per-block random streams, restated (CPU).

The reference draws Lanczos start vectors and randomized probes from
``np.random.default_rng(_block_seed(kind, node.id))`` (multiply.py:61-63,
compressors.py:303, :389, :424).  ``tests/np_random_ref.py`` restates SeedSequence, PCG64
and the ziggurat; the library's host generator (``hx_np_normals`` with device -1, the same
C++ code the kernels run, ``csrc/np_random.cuh``) must reproduce numpy bit for bit.
"""

import ctypes as C

import numpy as np
import pytest

import np_random_ref as R

SEEDS = [0, 1, 7, 12345, (7 << 24) ^ 99, (1 << 24) ^ 3548, 2**63 + 5, (2**45 << 24) ^ 3,
         2**100 + 17]


def _zig():
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tools"))
    import gen_ziggurat

    return gen_ziggurat.tables()


@pytest.mark.parametrize("seed", SEEDS)
def test_seed_sequence_and_pcg64(seed):
    assert R.seedseq_state(seed) == [int(x) for x in
                                     np.random.SeedSequence(seed).generate_state(4, np.uint64)]
    g = R.PCG64(seed)
    assert [g.next64() for _ in range(8)] == [int(x) for x in
                                              np.random.PCG64(seed).random_raw(8)]


@pytest.mark.parametrize("seed", SEEDS[:5])
def test_restated_normals(seed):
    ki, wi, fi = _zig()
    ref = np.random.default_rng(seed).standard_normal(3000)
    assert np.array_equal(R.normals(seed, 3000, ki, wi, fi), ref)


@pytest.mark.parametrize("seed", SEEDS)
def test_library_host_generator(seed):
    from paper_1805_08998_b200 import _lib

    n = 20000
    out = np.empty(n)
    lo, hi = seed & (2**64 - 1), seed >> 64
    _lib.check(_lib.lib().hx_np_normals(C.c_uint64(lo), C.c_uint64(hi), n,
                                        _lib.ptr(out, _lib.f64p), -1), "hx_np_normals")
    ref = np.random.default_rng(seed).standard_normal(n)
    assert np.array_equal(out, ref)

"""Kernel-level parity of the grouped DMMA GEMM against a NumPy fp64 reference.

Random tiles with several groups of terms: every operand layout (tile-contiguous and
k-contiguous), odd and even offsets / leading dimensions (16-byte and 8-byte copy paths),
odd k (segment packing), terms covering only part of the tile, ADD and SUMSQ epilogues.
"""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TERM = np.dtype([("a_off", "<i8"), ("b_off", "<i8"), ("a_ld", "<i4"), ("b_ld", "<i4"),
                 ("k", "<i4"), ("r_lo", "<i4"), ("c_lo", "<i4"), ("rows", "<i4"),
                 ("cols", "<i4"), ("a_buf", "u1"), ("b_buf", "u1"), ("a_kc", "u1"),
                 ("b_kc", "u1")])
TILE = np.dtype([("out_off", "<i8"), ("out_ld", "<i4"), ("row0", "<i4"), ("col0", "<i4"),
                 ("rows", "<i2"), ("cols", "<i2"), ("g_begin", "<i4"), ("g_end", "<i4"),
                 ("aux", "<i4"), ("out_buf", "u1"), ("mode", "u1"), ("pad", "u1", 2)])
GROUP = np.dtype([("t_begin", "<i4"), ("t_end", "<i4")])
NBUF = 10


def test_record_sizes():
    assert TERM.itemsize == 48 and TILE.itemsize == 40 and GROUP.itemsize == 8


def _operand(rng, buf, pos, idx_ext, k, kc):
    """Place a random (idx_ext x k) operand in buf at a random offset; returns (off, ld, M)."""
    ld = (idx_ext if kc == 0 else k) + int(rng.integers(0, 3))
    off = pos + int(rng.integers(0, 2))
    M = rng.standard_normal((idx_ext, k))
    i, kk = np.meshgrid(np.arange(idx_ext), np.arange(k), indexing="ij")
    buf[off + (i + kk * ld if kc == 0 else kk + i * ld)] = M
    return off, ld, M, off + (ld * k if kc == 0 else ld * idx_ext) + 4


@pytest.mark.parametrize("tile", [32, 64])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_grouped_gemm_matches_numpy(tile, seed):
    from paper_1805_08998_b200 import _lib

    rng = np.random.default_rng(seed)
    src = np.zeros(2_000_000)
    pos = 0
    terms, groups, tiles = [], [], []
    expected = []
    out = np.zeros(tile * tile * 8 + 64)
    n_tiles = 6
    for ti in range(n_tiles):
        rows = int(rng.integers(1, tile + 1)) if ti % 2 else tile
        cols = int(rng.integers(1, tile + 1)) if ti % 3 else tile
        row0, col0 = int(rng.integers(0, 1000)), int(rng.integers(0, 1000))
        exp = np.zeros((rows, cols))
        g0 = len(groups)
        for _ in range(int(rng.integers(1, 4))):
            t0 = len(terms)
            for _ in range(int(rng.integers(1, 6))):
                k = int(rng.integers(1, 41))
                a_kc, b_kc = int(rng.integers(0, 2)), int(rng.integers(0, 2))
                partial = rng.random() < 0.3
                r_lo = row0 - (int(rng.integers(-8, 9)) if partial else 0)
                c_lo = col0 - (int(rng.integers(-8, 9)) if partial else 0)
                trows = (rows + 16) if not partial else int(rng.integers(1, tile + 8))
                tcols = (cols + 16) if not partial else int(rng.integers(1, tile + 8))
                a_off, a_ld, P, pos = _operand(rng, src, pos, trows, k, a_kc)
                b_off, b_ld, Qt, pos = _operand(rng, src, pos, tcols, k, b_kc)
                terms.append((a_off, b_off, a_ld, b_ld, k, r_lo, c_lo, trows, tcols, 0, 0,
                              a_kc, b_kc))
                # expected contribution on the tile
                for i in range(rows):
                    ti_ = row0 + i - r_lo
                    if not 0 <= ti_ < trows:
                        continue
                    for j in range(cols):
                        tj = col0 + j - c_lo
                        if 0 <= tj < tcols:
                            exp[i, j] += P[ti_] @ Qt[tj]
            groups.append((t0, len(terms)))
        mode = int(rng.integers(0, 3))
        out_off = ti * tile * tile + 3
        if mode == 1:
            base = rng.standard_normal((rows, cols))
            for j in range(cols):
                out[out_off + j * tile: out_off + j * tile + rows] = base[:, j]
            exp = exp + base
        tiles.append((out_off, tile, row0, col0, rows, cols, g0, len(groups), ti, 1, mode,
                      (0, 0)))
        expected.append((out_off, rows, cols, exp, mode))
    t_arr = np.array(terms, dtype=TERM)
    l_arr = np.array(tiles, dtype=TILE)
    g_arr = np.array(groups, dtype=GROUP)
    bufs = (_lib.f64p * NBUF)()
    elems = np.zeros(NBUF, np.int64)
    bufs[0] = src.ctypes.data_as(_lib.f64p)
    elems[0] = src.size
    bufs[1] = out.ctypes.data_as(_lib.f64p)
    elems[1] = out.size
    sumsq = np.zeros(n_tiles)
    rc = _lib.lib().hx_debug_gemm(tile, t_arr.ctypes.data, len(t_arr), l_arr.ctypes.data,
                                  len(l_arr), g_arr.ctypes.data, len(g_arr), bufs,
                                  elems.ctypes.data_as(_lib.i64p), sumsq.ctypes.data_as(_lib.f64p),
                                  n_tiles)
    assert rc == 0, _lib.last_error()
    for ti, (off, rows, cols, exp, mode) in enumerate(expected):
        got = np.stack([out[off + j * tile: off + j * tile + rows] for j in range(cols)], axis=1)
        assert np.allclose(got, exp, rtol=1e-12, atol=1e-12 * max(1.0, np.abs(exp).max())), ti
        if mode == 2:
            assert abs(sumsq[ti] - np.sum(exp * exp)) <= 1e-10 * max(1.0, np.sum(exp * exp))


@pytest.mark.parametrize("tile", [64, -64])
def test_grouped_gemm_many_tiles(tile):
    """Thousands of tiles (more than one per resident CTA: the persistent kernel walks
    several tiles per CTA and wraps its stage ring many times), random terms in every
    layout, partial coverage, empty tiles, STORE / ADD / SUMSQ epilogues; -64 runs the
    short-K configuration of the term-formation batches."""
    from paper_1805_08998_b200 import _lib

    T = 64
    rng = np.random.default_rng(11)
    n_tiles = 3000
    src = np.zeros(40_000_000)
    pos = 0
    terms, groups, tiles, checks = [], [], [], []
    out = np.zeros(n_tiles * T * T + 8)
    for ti in range(n_tiles):
        rows = T if rng.random() < 0.7 else int(rng.integers(1, T + 1))
        cols = T if rng.random() < 0.7 else int(rng.integers(1, T + 1))
        exp = np.zeros((rows, cols))
        g0 = len(groups)
        n_groups = 0 if rng.random() < 0.03 else int(rng.integers(1, 3))
        for _ in range(n_groups):
            t0 = len(terms)
            for _ in range(int(rng.integers(1, 4))):
                k = int(rng.integers(1, 40))
                a_kc, b_kc = int(rng.integers(0, 2)), int(rng.integers(0, 2))
                partial = rng.random() < 0.25
                dr = int(rng.integers(-8, 9)) if partial else 0
                dc = int(rng.integers(-8, 9)) if partial else 0
                trows = rows if not partial else int(rng.integers(1, T + 8))
                tcols = cols if not partial else int(rng.integers(1, T + 8))
                a_off, a_ld, P, pos = _operand(rng, src, pos, trows, k, a_kc)
                b_off, b_ld, Qt, pos = _operand(rng, src, pos, tcols, k, b_kc)
                # tile (i, j) <- term row i + dr, col j + dc  (r_lo = row0 - dr)
                terms.append((a_off, b_off, a_ld, b_ld, k, -dr, -dc, trows, tcols, 0, 0,
                              a_kc, b_kc))
                i0, i1 = max(0, -dr), min(rows, trows - dr)
                j0, j1 = max(0, -dc), min(cols, tcols - dc)
                if i1 > i0 and j1 > j0:
                    exp[i0:i1, j0:j1] += P[i0 + dr:i1 + dr] @ Qt[j0 + dc:j1 + dc].T
            groups.append((t0, len(terms)))
        mode = int(rng.integers(0, 3))
        out_off = ti * T * T
        if mode == 1:
            base = rng.standard_normal((rows, cols))
            out[out_off:out_off + T * cols].reshape(cols, T)[:, :rows] = base.T
            exp = exp + base
        tiles.append((out_off, T, 0, 0, rows, cols, g0, len(groups), ti, 1, mode, (0, 0)))
        checks.append((out_off, rows, cols, exp, mode))
    assert pos < src.size
    t_arr = np.array(terms, dtype=TERM)
    l_arr = np.array(tiles, dtype=TILE)
    g_arr = np.array(groups if groups else [(0, 0)], dtype=GROUP)
    bufs = (_lib.f64p * NBUF)()
    elems = np.zeros(NBUF, np.int64)
    bufs[0] = src.ctypes.data_as(_lib.f64p)
    elems[0] = src.size
    bufs[1] = out.ctypes.data_as(_lib.f64p)
    elems[1] = out.size
    sumsq = np.zeros(n_tiles)
    rc = _lib.lib().hx_debug_gemm(tile, t_arr.ctypes.data, len(t_arr), l_arr.ctypes.data,
                                  len(l_arr), g_arr.ctypes.data, len(g_arr), bufs,
                                  elems.ctypes.data_as(_lib.i64p), sumsq.ctypes.data_as(_lib.f64p),
                                  n_tiles)
    assert rc == 0, _lib.last_error()
    for ti, (off, rows, cols, exp, mode) in enumerate(checks):
        got = out[off:off + T * cols].reshape(cols, T)[:, :rows].T
        assert np.allclose(got, exp, rtol=1e-12, atol=1e-12 * max(1.0, np.abs(exp).max())), ti
        if mode == 2:
            assert abs(sumsq[ti] - np.sum(exp * exp)) <= 1e-10 * max(1.0, np.sum(exp * exp))

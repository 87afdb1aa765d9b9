"""GPU matrix-free compressors (csrc/iterative.cuh) against the unmodified reference.

``tests/golden/compressors.npz`` holds the reference's ``compress`` outputs
(compressors.py:441-452) on its own test operators (a geometric-decay matrix and an exact
rank-7 one; reference test_compressors.py:11-23) for every tag and three policies, with
CompressorKind seed 7 and the CountingMap totals.  ``hx_debug_compress`` runs one block
through the same device route as the product (aca: the cross iteration then
truncate(eps/2); bilanczos: GKL then the core SVD; randomized: adaptive or blocked finder)
with the per-block numpy stream default_rng((0 << 24) ^ 7) = default_rng(7).
"""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TAG = {"aca": 0, "bilanczos": 1, "randomized": 2}


def compress(a, tag, policy, eps=0.0, k_max=0, q=1, seed=0, node=7):
    from paper_1805_08998_b200 import _lib

    a = np.asfortranarray(a, dtype=np.float64)
    m, n = a.shape
    mu = min(m, n)
    left = np.zeros(m * mu)
    right = np.zeros(n * mu)
    info = np.zeros(3, np.int32)
    flat = np.ascontiguousarray(a.T).ravel()  # column-major
    _lib.check(_lib.lib().hx_debug_compress(TAG[tag], policy, eps, k_max, q, C.c_uint64(seed),
                                            node, m, n, _lib.ptr(flat, _lib.f64p),
                                            _lib.ptr(left, _lib.f64p),
                                            _lib.ptr(right, _lib.f64p),
                                            _lib.ptr(info, _lib.i32p)), "hx_debug_compress")
    r = int(info[0])
    return (left[:m * r].reshape(r, m).T, right[:n * r].reshape(r, n).T, r, int(info[1]),
            int(info[2]))


@pytest.mark.parametrize("seed", [0, 7, (3 << 24) ^ 1001, 2**64 + 9])
def test_device_normals_match_numpy(seed):
    from paper_1805_08998_b200 import _lib

    n = 50000
    out = np.empty(n)
    _lib.check(_lib.lib().hx_np_normals(C.c_uint64(seed & (2**64 - 1)), C.c_uint64(seed >> 64),
                                        n, _lib.ptr(out, _lib.f64p), 0), "hx_np_normals")
    assert np.array_equal(out, np.random.default_rng(seed).standard_normal(n))


@pytest.mark.parametrize("mat", ["decay", "lowr"])
@pytest.mark.parametrize("pol", ["eps1e-6", "eps1e-10", "fixed5"])
@pytest.mark.parametrize("tag", ["aca", "bilanczos", "randomized"])
def test_compressor_matches_reference(golden, mat, pol, tag):
    g = golden("compressors.npz")
    a = g[mat]
    key = f"{mat}/{pol}/{tag}"
    ref = g[f"{key}/left"] @ g[f"{key}/right"].T
    count, deg = (int(x) for x in g[f"{key}/count"])
    if pol == "fixed5":
        left, right, r, d, mv = compress(a, tag, 1, k_max=5)
    else:
        left, right, r, d, mv = compress(a, tag, 0, eps=float(pol[3:]))
    assert r == g[f"{key}/left"].shape[1], (r, g[f"{key}/left"].shape)
    assert (mv, d) == (count, deg)
    scale = np.linalg.norm(a)
    assert np.linalg.norm(left @ right.T - ref) <= 1e-10 * scale


@pytest.mark.parametrize("tag", ["aca", "bilanczos", "randomized"])
def test_zero_and_rank_one_blocks(tag):
    """A zero block: ACA samples every row as zero (certified, not degraded), Lanczos
    probes three times, the range finder stops at once; all return rank 0."""
    z = np.zeros((40, 30))
    left, right, r, d, mv = compress(z, tag, 0, eps=1e-8)
    assert r == 0 and d == 0
    if tag == "aca":
        assert mv == 40  # one row per sampled row, no column
    u = np.linspace(1, 2, 40)[:, None] * np.linspace(-1, 1, 30)[None, :]
    left, right, r, d, mv = compress(u, tag, 0, eps=1e-8)
    assert r >= 1
    assert np.linalg.norm(left @ right.T - u) <= 1e-10 * np.linalg.norm(u)

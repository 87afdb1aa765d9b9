"""The five BASELINE configurations (BASELINE.json ``configs``).

Synthetic, seeded inputs exactly as specified: points from ``np.random.default_rng(seed)``
(uniform square / cube, or normalised Gaussians for the unit sphere), unit quadrature
weights, operands assembled by ACA (on the GPU, ``assembly.assemble_hmatrix``).
"""

from __future__ import annotations

import numpy as np

from .assembly import assemble_hmatrix
from .clustering import build_block_cluster_tree, build_cluster_tree
from .lowrank import EpsRank

CONFIGS = {
    1: dict(n=2048, geometry="square", ka="exp", kb=None, n_min=32, eta=0.8, eps_a=1e-8,
            tol=1e-6),
    2: dict(n=32768, geometry="sphere", ka="gauss0.1", kb=None, n_min=64, eta=0.8,
            eps_a=1e-8, tol=1e-6),
    3: dict(n=131072, geometry="cube", ka="exp0.5", kb="inv", n_min=64, eta=1.0, eps_a=1e-8,
            tol=1e-8),
    4: dict(n=1048576, geometry="square", ka="exp", kb=None, n_min=64, eta=0.8, eps_a=1e-6,
            tol=1e-4),
    5: dict(n=262144, geometry="cube", ka="exp", kb=None, n_min=128, eta=1.5, eps_a=1e-12,
            tol=1e-10),
}

NAMES = {
    1: "cfg1: n=2048 [0,1]^2 exp(-r) leaf32 eta0.8 ACA1e-8, C=A*A tol1e-6",
    2: "cfg2: n=32768 S^2 exp(-r^2/0.1) leaf64 eta0.8 ACA1e-8, C=A*A tol1e-6",
    3: "cfg3: n=131072 cube A=exp(-r/0.5) B=1/(r+h) leaf64 eta1.0 ACA1e-8, C=A*B tol1e-8",
    4: "cfg4: n=1048576 [0,1]^2 exp(-r) leaf64 eta0.8 ACA1e-6, C=A*A tol1e-4",
    5: "cfg5: n=262144 cube exp(-r) leaf128 eta1.5 ACA1e-12, C=A*A tol1e-10",
}


def make_points(c, seed=0):
    rng = np.random.default_rng(seed)
    n = c["n"]
    if c["geometry"] == "square":
        return rng.uniform(0, 1, (n, 2))
    if c["geometry"] == "cube":
        return rng.uniform(0, 1, (n, 3))
    g = rng.standard_normal((n, 3))
    return g / np.linalg.norm(g, axis=1, keepdims=True)


def build_operands(c, seed=0, device=0):
    pts = make_points(c, seed)
    bct = build_block_cluster_tree(build_cluster_tree(pts, c["n_min"]), c["eta"])
    h = c["n"] ** (-1.0 / 3.0)
    A = assemble_hmatrix(c["ka"], bct, EpsRank(c["eps_a"]), pts, h=h, device=device)
    B = A if c["kb"] is None else assemble_hmatrix(c["kb"], bct, EpsRank(c["eps_a"]), pts,
                                                   h=h, device=device)
    return bct, A, B

"""CPU checks of bench.py's measurement pieces: the canonical work of the product's units
adds up to the whole product's (so a stratified unit sample prices the whole product),
the stratified ratio estimator, and the CPU reference arm runs without loading any part
of the GPU library."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_units_partition_canonical_work(golden):
    import bench
    import paper_1805_08998_b200 as hx
    from oracle import hmat_oracle as O
    from paper_1805_08998_b200 import _lib, hmatrix, multiply

    g = golden("cfg1.npz")
    n, n_min, eta, eps_a, tol = g["params"]
    pts = g["points"]
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, int(n_min)), eta)
    obt = O.BlockTreeO(O.ClusterTreeO(pts, int(n_min)), eta)
    A = hx.HMatrix(bct, O.assemble_o("exp", obt, O.Eps(eps_a), pts).data)
    _, d = hmatrix.pack_operand(A)
    rank_of = dict(zip(g["aca/ids"].tolist(), g["aca/ranks"].tolist()))
    ta = hmatrix.tree_arrays(bct)
    tile = multiply.plan_tile(bct)

    def work(mask):
        p = _lib.Plan(ta, d, d, mask, tile)
        lv = p.leaves()
        ph = bench.canonical_phases(p.info, lv, np.array([rank_of[int(b)] for b in lv["ids"]]))
        p.close()
        return ph

    whole = work(None)
    arr = hmatrix.block_arrays(bct)
    leaf = arr.kind_code != 0
    units = multiply.chunk_units(bct)
    covered = np.zeros(arr.n_nodes, bool)
    tot = {"F": 0.0, "B": 0.0}
    for b0, b1, _ in units:
        m = np.zeros(arr.n_nodes, np.uint8)
        m[b0:b1] = leaf[b0:b1]
        assert not covered[b0:b1].any()
        covered[b0:b1] = True
        u = work(m)
        tot["F"] += u["F"]
        tot["B"] += u["B"]
    assert covered[leaf].all()
    assert abs(tot["F"] - whole["F"]) <= 1e-9 * whole["F"]
    assert abs(tot["B"] - whole["B"]) <= 1e-9 * whole["B"]
    # phase split adds up; the roofline time is positive and below the sum of both bounds
    assert abs(sum(whole[k]["F"] for k in ("form", "near", "far")) - whole["F"]) < 1.0
    t = bench.roofline_time(whole, 37.1, 6500.0)
    assert 0 < t <= whole["F"] / 37.1e12 + whole["B"] / 6.5e12


def test_stratified_estimator_recovers_rate():
    """Units whose run time is exactly F / rate: the estimate is that rate, whatever the
    strata and draws."""
    import bench

    rng = np.random.default_rng(3)
    F = rng.lognormal(20, 1.5, 400)
    b0 = np.arange(400) * 2
    table = {"F": F, "b0": b0, "b1": b0 + 2, "F_total": F.sum()}
    kind = np.ones(800, np.int8)
    clock = [0.0]
    s = bench.UnitSampler(table, kind, strata=8, seed=0, clock=lambda: clock[0])
    rate = 7.5e9

    def run(only):
        u = min(only) // 2
        clock[0] += F[u] / rate

    s.step(run, 50 * F.mean() / rate)
    v, T = s.estimate()
    assert abs(v * 1e9 - rate) <= 1e-9 * rate
    assert abs(T - F.sum() / rate) <= 1e-9 * T
    assert s.units > 0


@pytest.mark.slow
def test_reference_arm_loads_no_native_library(tmp_path):
    if not os.path.exists(os.path.join(ROOT, "bench_data", "cfg1_aca_units.npz")):
        pytest.skip("unit table for cfg1 not generated")
    env = dict(os.environ, OPENBLAS_NUM_THREADS="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl",
                          "reference", "--config", "1", "--steps", "1", "--warmup", "1",
                          "--cpu-budget", "0.5"], capture_output=True, text=True, env=env,
                         timeout=600, cwd=tmp_path)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["native_libs_loaded"] == []
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["compressor"] == "aca"
    assert line["cpu_baseline"]["kind"] == "port"

"""Benchmark of the tolerance-controlled H x H product (BASELINE.json metric).

One step = one full product C = A*B on the bench workload (default: BASELINE config 2,
n=32768 on S^2, Gaussian kernel, leaf 64, eta 0.8, ACA 1e-8 operands, tol 1e-6, the
reference CLI's default compressor ``aca``), operands resident in HBM: host-side term-list
planning + all device phases, bracketed by CUDA events on the product stream (barrier +
synchronize on both sides; max over ranks).

value  = canonical FP64 work of the product (SURVEY 8(d) min-route model) / step time,
         in GFLOP/s, whole job.
e2e    = the same through the public API with host operands: H2D of the operand pool,
         the product, D2H of every output block and construction of the HMatrix.
Also: the whole product against its phase-wise roofline, the relative error (the
reference's estimator on the GPU), the other compressor (``--alt-tag``) on the same
operands, and the CPU baseline (the oracle port on a stratified sample of units).
Multi-GPU (torchrun): output subtrees are partitioned over ranks (priced once on rank 0),
operand pools replicated from rank 0 by an NCCL broadcast; no reduction (strong scaling).

--impl reference: the reference algorithm (the NumPy restatement in oracle/; the reference
is pure Python and cannot travel to the GPU box) on the host cores, on operands assembled
by the port's own ACA, timed on a stratified sample of the product's units and priced by
the committed per-unit canonical work table (bench_data/, tools/unit_table.py); no part of
the GPU library is loaded.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_DMMA_PEAK_TFLOPS = 37.1   # profiles/r01_fp64_peak.txt (measured, this pool's B200)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks sampling
class Clocks:
    def __init__(self, device):
        self.proc = None
        self.path = None
        self.device = device

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:  # pragma: no cover
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ canonical work
def canonical_phases(info, leaves, ranks):
    """canonical F (flops) and B (bytes) of a plan's product given its leaves
    and the far ranks, whole and per phase (term formation, near leaves, far leaves at the
    cheapest of the dense / factor / sketch routes)."""
    far = leaves["kind"] == 1
    m = leaves["m"][far].astype(float)
    n = leaves["n"][far].astype(float)
    K = leaves["K"][far].astype(float)
    fdd = leaves["fdd"][far]
    edd = leaves["edd"][far]
    r = np.asarray(ranks)[far].astype(float)
    mu = np.minimum(m, n)
    ell = np.minimum(r + 8, mu)
    f_dense = fdd + 2 * m * n * K + 14 * m * n * mu + 8 * mu ** 3 + 2 * (m + n) * mu * r
    b_dense = 8 * (K * (m + n) + edd + 2 * m * n + (m + n) * r)
    f_fact = np.where((fdd == 0) & (K < mu),
                      2 * m * K ** 2 + 2 * n * K ** 2 - (4 / 3) * K ** 3 + 2 * K ** 3 + 22 * K ** 3
                      + 2 * (m + n) * K * r, np.inf)
    b_fact = 8 * (2 * K * (m + n) + (m + n) * r)
    f_sk = (2 * ell * (2 * K * (m + n) + 2 * edd) + 2 * m * ell ** 2 + 14 * n * ell ** 2
            + 8 * ell ** 3 + 2 * (m + n) * ell * r)
    b_sk = 8 * (2 * (K * (m + n) + edd) + 2 * ell * (m + n))
    fs = np.stack([f_dense, f_fact, f_sk])
    bs = np.stack([b_dense, b_fact, b_sk])
    pick = np.argmin(fs, axis=0)
    cols = np.arange(len(m))
    out = {"form": {"F": float(info.flops_form), "B": float(info.bytes_form)},
           "near": {"F": float(info.flops_near), "B": float(info.bytes_near)},
           "far": {"F": float(fs[pick, cols].sum()), "B": float(bs[pick, cols].sum())}}
    out["F"] = sum(out[k]["F"] for k in ("form", "near", "far"))
    out["B"] = sum(out[k]["B"] for k in ("form", "near", "far"))
    return out


def canonical_work(info, leaves, ranks):
    ph = canonical_phases(info, leaves, ranks)
    return ph["F"], ph["B"]


def roofline_time(ph, p64_tflops, bw_gbs):
    """Phase-wise roofline time of the whole product: sum over phases of max(F/P, B/BW)."""
    return sum(max(ph[k]["F"] / (p64_tflops * 1e12), ph[k]["B"] / (bw_gbs * 1e9))
               for k in ("form", "near", "far"))


# ------------------------------------------------------------------ partition
def lpt_partition(cost, world):
    """Longest-processing-time greedy: leaf index -> rank."""
    order = np.argsort(-cost, kind="stable")
    load = np.zeros(world)
    owner = np.zeros(len(cost), dtype=np.int64)
    for i in order:
        r = int(np.argmin(load))
        owner[i] = r
        load[r] += cost[i]
    return owner, load


def leaf_costs(leaves):
    from paper_1805_08998_b200.distributed import leaf_costs as lc
    return lc(leaves)


# ------------------------------------------------------------------ CPU reference sample
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:  # pragma: no cover
        pass
    return "unknown CPU"


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max(int(i.get("num_threads", 1)) for i in threadpool_info()
                   if i.get("user_api") == "blas")
    except Exception:  # pragma: no cover
        return int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))


def unit_table(cfg_id, tag):
    """The committed per-unit canonical work table (tools/unit_table.py), or None."""
    path = os.path.join(ROOT, "bench_data", f"cfg{cfg_id}_{tag}_units.npz")
    if not os.path.exists(path):
        return None
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


class UnitSampler:
    """Stratified sample of the product's units (subtrees at the first block level holding
    a far leaf: they share no work, their canonical work adds up to the product's).

    The units are split into ``strata`` groups of equal total canonical work (ordered by
    unit work); each step runs whole units through the reference algorithm (the oracle's
    ``hmult_new_o`` restricted to the unit's leaves: the same DFS, restrict and compress
    calls, plus the short descent from the root to the unit), one unit drawn at random from
    each stratum in turn, until the step's time budget is spent.  The product time is
    estimated stratum by stratum: stratum work x measured seconds per flop of its sampled
    units (a stratified ratio estimator); GFLOP/s = canonical work / that time."""

    def __init__(self, table, kind, strata=16, seed=0, clock=time.perf_counter):
        self.clock = clock
        self.F = np.asarray(table["F"], float)
        self.b0 = np.asarray(table["b0"])
        self.b1 = np.asarray(table["b1"])
        self.F_total = float(table["F_total"])
        self.kind = kind
        order = np.argsort(self.F, kind="stable")
        cum = np.cumsum(self.F[order]) / max(self.F.sum(), 1e-300)
        cut = np.searchsorted(cum, np.arange(1, strata) / strata)
        self.strata = [g for g in np.split(order, cut) if g.size]
        self.FH = np.array([self.F[g].sum() for g in self.strata])
        self.rng = np.random.default_rng(seed)
        self.t = np.zeros(len(self.strata))
        self.f = np.zeros(len(self.strata))
        self.units = 0
        self.cursor = 0

    def leaves(self, u):
        return {b for b in range(int(self.b0[u]), int(self.b1[u])) if self.kind[b] != 0}

    def step(self, run, budget_s, record=True):
        """Run units for about ``budget_s`` seconds; ``run(leaf set)`` is the timed call."""
        spent = 0.0
        while spent < budget_s:
            h = self.cursor % len(self.strata)
            self.cursor += 1
            u = int(self.rng.choice(self.strata[h]))
            only = self.leaves(u)
            t0 = self.clock()
            run(only)
            dt = self.clock() - t0
            spent += dt
            if record:
                self.t[h] += dt
                self.f[h] += self.F[u]
                self.units += 1
        return spent

    def estimate(self):
        """(GFLOP/s, estimated seconds of the whole product)."""
        seen = self.f > 0
        rate = self.f[seen].sum() / self.t[seen].sum()
        T = float(np.sum(np.where(seen, self.FH * self.t / np.maximum(self.f, 1e-300),
                                  self.FH / rate)))
        return self.F_total / T / 1e9, T

    def describe(self):
        return (f"{self.units} units (subtrees at the first far level) drawn from "
                f"{len(self.strata)} equal-work strata of the {len(self.F)} units, "
                f"{self.t.sum():.1f} s timed; whole-product time by the stratified ratio "
                f"estimator")


def oracle_operand(H):
    """The GPU arm's operand as an oracle HMatO (the same blocks, numpy views)."""
    from oracle import hmat_oracle as O

    data = {}
    for b, p in H.data.items():
        data[b] = O.LR(np.ascontiguousarray(p.left), np.ascontiguousarray(p.right)) \
            if hasattr(p, "left") else np.ascontiguousarray(p)
    return data


def cpu_run(oa, ob, tol, tag):
    from oracle import hmat_oracle as O

    def run(only):
        O.hmult_new_o(oa, ob, O.Eps(tol), tag, only=only)
    return run


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    # the reference CLI's default compressor (cli.py:57); both arms run the same tag
    ap.add_argument("--tag", default="aca")
    ap.add_argument("--alt-tag", default="dense-svd",
                    help="second compressor timed on the same operands ('' to skip)")
    ap.add_argument("--cpu-budget", type=float, default=0.0,
                    help="seconds of CPU work per reference step (0: fit the run in ~2.5 min)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return bench_reference(args, rank, world)
    return bench_ours(args, rank, world, local)


def mapped_native_libs():
    """Shared objects of this repo mapped into the process (evidence for the CPU arm)."""
    out = set()
    try:
        for line in open("/proc/self/maps"):
            path = line.split()[-1] if len(line.split()) >= 6 else ""
            if path.startswith(ROOT) and ".so" in path:
                out.add(os.path.relpath(path, ROOT))
    except OSError:  # pragma: no cover
        pass
    return sorted(out)


def step_budget(args):
    """Seconds of CPU work per step: the whole --warmup W --steps K run within ~2.5 min."""
    if args.cpu_budget > 0 and args.impl == "reference":
        return args.cpu_budget
    return float(np.clip(150.0 / max(args.warmup + args.steps, 1), 2.0, 20.0))


def bench_reference(args, rank, world):
    """The reference algorithm on the host cores: the oracle port of hmult_new (NumPy /
    OpenBLAS, every host thread BLAS uses), on operands assembled by the port's own ACA
    (assembly is setup, as in cli.py:150-158), timed on a stratified sample of the
    product's units; nothing of the GPU library is loaded."""
    if rank != 0:
        return 0
    from oracle import hmat_oracle as O
    from paper_1805_08998_b200.configs import CONFIGS, NAMES  # plain dicts (no library load)

    c = CONFIGS[args.config]
    table = unit_table(args.config, args.tag)
    if table is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"no unit table bench_data/cfg{args.config}_{args.tag}_units.npz"}))
        return 0
    t_setup = time.perf_counter()
    pts = O.make_points(c)
    bt = O.BlockTreeO(O.ClusterTreeO(pts, c["n_min"]), c["eta"])
    h = c["n"] ** (-1.0 / 3.0)
    oa = O.assemble_parallel_o(c["ka"], bt, O.Eps(c["eps_a"]), pts, h=h)
    ob = oa if c["kb"] is None else O.assemble_parallel_o(c["kb"], bt, O.Eps(c["eps_a"]), pts,
                                                          h=h)
    setup_s = time.perf_counter() - t_setup
    sampler = UnitSampler(table, bt.kind)
    run = cpu_run(oa, ob, c["tol"], args.tag)
    budget = step_budget(args)
    for i in range(args.warmup + args.steps):
        sampler.step(run, budget, record=i >= args.warmup)
    v, T = sampler.estimate()
    threads = blas_threads()
    line = {
        "impl": "reference", "metric": "hxh_product_fp64_gflops", "value": v,
        "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sampler.t.sum() / max(args.steps, 1),
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE point cloud, operands assembled by the port's ACA)",
        "config": {"workload": NAMES[args.config], "compressor": args.tag},
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": threads, "kind": "port",
                         "cpu": cpu_model(), "host_cpus": os.cpu_count(),
                         "sample": f"reference algorithm (oracle NumPy port of hmult_new, "
                                   f"{args.tag} compressor) on {sampler.describe()}; "
                                   f"{budget:.1f} s per step"},
        "product_s_estimate": T, "canonical_gflop": float(table["F_total"]) / 1e9,
        "ms_per_step_note": "CPU seconds of one step's unit sample; product_s_estimate is "
                            "the whole product's estimated time",
        "setup_s": setup_s, "native_libs_loaded": mapped_native_libs(),
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def bench_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200 import _lib, configs, distributed, hmatrix, multiply

    os.environ.setdefault("HX_MALLOPT", "1")  # see _lib._tune_host_allocator
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = configs.CONFIGS[args.config]
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind(args.tag), policy=hx.EpsRank(c["tol"]))
    pts = configs.make_points(c)
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, c["n_min"]), c["eta"])
    h = c["n"] ** (-1.0 / 3.0)
    bcast_ms, bcast_bytes = [], []  # NCCL operand broadcasts (setup, outside the timed step)

    def operand(kern):
        if world == 1:
            return hx.assemble_hmatrix(kern, bct, hx.EpsRank(c["eps_a"]), pts, h=h, device=local)
        # rank 0 assembles; the packed pool goes to every rank by an NCCL broadcast
        # (distributed.broadcast_operand: the data plane of hmult_new_spmd)
        H = hx.assemble_hmatrix(kern, bct, hx.EpsRank(c["eps_a"]), pts, h=h, device=local) \
            if rank == 0 else None
        torch.cuda.synchronize()
        t0b = time.perf_counter()
        H = distributed.broadcast_operand(H, bct, 0, None, device=local)
        torch.cuda.synchronize()
        bcast_ms.append(1e3 * (time.perf_counter() - t0b))
        bcast_bytes.append(8 * max(H._hx_device[2], 1))
        return H

    t_setup = time.time()
    A = operand(c["ka"])
    B = A if c["kb"] is None else operand(c["kb"])
    _, dA = multiply.operand_directory(A)
    _, dB = multiply.operand_directory(B)
    pool_gb = 8 * sum(H._hx_device[2] for H in ({id(A): A, id(B): B}.values())) / 1e9
    mask = None
    if world > 1:
        # the partition is priced once (measured planning times) on rank 0 and shipped
        masks = [distributed.partition(A, B, world, tag=args.tag)[0] if rank == 0 else None]
        dist.broadcast_object_list(masks, src=0)
        mask = masks[0][rank]
    setup_s = time.time() - t_setup
    # tensor-core work of this rank's plan (outside the timed region)
    mma = np.zeros(6)
    wp = _lib.Plan(hmatrix.tree_arrays(bct), dA, dA if B is A else dB, mask,
                   multiply.plan_tile(bct), flags=multiply.implicit_flags(None, args.tag))
    _lib.check(_lib.lib().hx_plan_mma_flops(wp.h, _lib.ptr(mma, _lib.f64p)), "mma flops")
    wp.close()

    stream = torch.cuda.current_stream()

    def step():
        # operands resident, output blocks stay in HBM (the e2e leg below fetches them)
        return multiply.multiply_device(A, B, cfg, device=local, leaf_mask=mask, fetch=False)

    for _ in range(args.warmup):
        C = step()
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    launches = 0
    for _ in range(args.steps):
        C = step()
        launches += C.report.launches
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    # canonical work of the whole product (all ranks' leaves)
    lv = C.plan_leaves
    ph = canonical_phases(C.plan_info, lv, C.leaf_rank)
    ranks_all = None
    if world > 1:
        full = _lib.Plan(hmatrix.tree_arrays(bct), dA, dA if B is A else dB, None,
                         multiply.plan_tile(bct))
        lv_all = full.leaves()
        # far ranks of every leaf: gather owned ranks
        mine = dict(zip(lv["ids"].tolist(), C.leaf_rank.tolist()))
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        allr = {}
        for g in gathered:
            allr.update(g)
        ranks_all = np.array([allr[int(b)] for b in lv_all["ids"]])
        ph = canonical_phases(full.info, lv_all, ranks_all)
    F_tot, B_tot = ph["F"], ph["B"]
    value = F_tot / (ms_max * 1e-3) / 1e9

    # roofline of the dominant kernel: the materialization launch of grouped_gemm_kernel
    # (one launch per step, FP64 DMMA-bound); algorithmic flops = exact useful products
    # sum over tiles and terms of 2 * rows * cols * k (no padding), from the plan
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6552.3))
    info = C.plan_info
    # the timed steps overlap chunks on two streams, so their per-phase event times include
    # contention: the kernel durations come from one more product after the timed region,
    # run without overlap (same plan, same kernels), events on the launching stream
    for _ in range(2):  # the second run reuses the first one's device buffers
        Ci = multiply.multiply_device(A, B, cfg, device=local, leaf_mask=mask, fetch=False,
                                      chunks=C.report.chunks, overlap=False)
    ri = Ci.report
    iso = {"plan_host": ri.plan_ms, "upload": ri.upload_ms, "form": ri.form_ms,
           "materialize": ri.materialize_ms, "recompress": ri.recompress_ms,
           "device_total": ri.device_ms, "chunks": ri.chunks}
    mat_s = ri.materialize_ms * 1e-3
    form_ms_iso = ri.form_ms
    mat_tflops = mma[5] / mat_s / 1e12 if mat_s > 0 else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "mat_kernel_traffic.json")) as f:
            tj = json.load(f)
        if tj.get("config") == args.config:
            traffic = tj["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        pass
    form_s = form_ms_iso * 1e-3
    form_gbs = info.bytes_form / form_s / 1e9 if form_s > 0 else 0.0
    roofline = {"bound": "tensor", "achieved": mat_tflops, "peak": FP64_DMMA_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": mat_tflops / FP64_DMMA_PEAK_TFLOPS,
                "traffic": traffic,
                "kernel": "grouped_gemm_ws_kernel<Ws64> materialization launches (per product)",
                "algorithmic_flops_per_launch": mma[5],
                "issued_flops_per_launch": mma[2],
                "peak_source": "FP64 DMMA measured on this pool's B200 (tools/fp64_peak.cu, "
                               "profiles/r01_fp64_peak.txt); MEASURED_PEAKS.json has no FP64 "
                               "entry",
                "formation_phase": {"bound": "hbm", "achieved_gbs": form_gbs, "peak_gbs": hbm,
                                    "frac": form_gbs / hbm,
                                    "note": "canonical term-formation bytes (SURVEY 8(d)) / "
                                            "formation phase time"},
                "fp64_tflops_whole_product": value / 1e3,
                "fp64_frac_whole_product": value / 1e3 / FP64_DMMA_PEAK_TFLOPS}
    # the whole product against its phase-wise canonical roofline
    t_roof = roofline_time(ph, FP64_DMMA_PEAK_TFLOPS, hbm)
    roofline["whole_product"] = {
        "t_roof_ms": t_roof * 1e3, "frac": t_roof / (ms_max * 1e-3),
        "frac_e2e": None,
        "phases": {k: {"gflop": ph[k]["F"] / 1e9, "gbytes": ph[k]["B"] / 1e9,
                       "t_roof_ms": 1e3 * max(ph[k]["F"] / (FP64_DMMA_PEAK_TFLOPS * 1e12),
                                              ph[k]["B"] / (hbm * 1e9))}
                   for k in ("form", "near", "far")},
        "note": "T_roof = sum over phases of max(F / P64, B / HBM) with the canonical "
                "min-route work model; frac = T_roof / ms_per_step"}
    # the other compressor on the same operands (device-resident, same timing)
    alt = None
    if args.alt_tag and args.alt_tag != args.tag:
        cfg2 = hx.MultiplyConfig(compressor=hx.CompressorKind(args.alt_tag),
                                 policy=hx.EpsRank(c["tol"]))
        for _ in range(max(args.warmup, 2)):
            Ca = multiply.multiply_device(A, B, cfg2, device=local, leaf_mask=mask, fetch=False)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            Ca = multiply.multiply_device(A, B, cfg2, device=local, leaf_mask=mask, fetch=False)
        e1.record(stream)
        torch.cuda.synchronize()
        ta_ = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64,
                           device="cuda")
        if world > 1:
            dist.all_reduce(ta_, op=dist.ReduceOp.MAX)
        pa_ = canonical_phases(Ca.plan_info, Ca.plan_leaves, Ca.leaf_rank) if world == 1 else None
        alt = {"compressor": args.alt_tag, "ms_per_step": float(ta_.item()),
               "value": (pa_["F"] / (float(ta_.item()) * 1e-3) / 1e9) if pa_ else None,
               "max_far_rank": Ca.report.max_far_rank}
    # relative error of the product against A*B, through the GPU H-matrix x block
    # products: the reference's estimator (two-sided block subspace iteration on C - A B,
    # multiply.py:266-294) over ||C||_F, and an unbiased probe estimate
    rel_err = None
    if world == 1 and not args.no_e2e:
        from paper_1805_08998_b200 import matvec
        t_err = time.perf_counter()
        Cr = multiply.multiply_device(A, B, cfg, device=local, leaf_mask=mask)
        est = matvec.estimate_product_error(A, B, Cr, device=local)
        fro = hx.frobenius_norm(Cr)
        probe, _ = matvec.product_error(Cr, A, B, probes=16, device=local)
        rel_err = {"value": est / fro, "estimator": "estimate_product_error (10 "
                   "iterations, block 100) / ||C||_F", "probe16": probe,
                   "tol": c["tol"], "seconds": time.perf_counter() - t_err}
        del Cr

    # e2e through the public API with host operands (last GPU phase: the device-resident
    # pools are released first, the uploads need their room on the large configs)
    e2e = None
    if not args.no_e2e:
        pa, _ = multiply._host_directory(A)
        pb = pa if B is A else multiply._host_directory(B)[0]
        h2d = 8 * (pa.size + (0 if B is A else pb.size))
        for H in (A, B):
            for name in ("_hx_pool", "_hx_device", "_hx_keep"):
                H.__dict__.pop(name, None)
        torch.cuda.empty_cache()
        for _ in range(2):  # warm-up: page-locked result buffers enter the reuse cache
            del_me = multiply.multiply_device(A, B, cfg, device=local, leaf_mask=mask,
                                              device_operands=False)
            del del_me
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d2h = 0
        Ce = None
        for _ in range(args.steps):
            # the previous step's result is released first (as a caller replacing it
            # would), so its page-locked buffers are reused instead of pinning new ones
            Ce = None
            Ce = multiply.multiply_device(A, B, cfg, device=local, leaf_mask=mask,
                                          device_operands=False)
            # bytes of the result buffers copied back (every far factor and near block);
            # the HMatrix builds its leaf views over them on access
            d2h = 8 * int(Ce.report.out_elems)
        torch.cuda.synchronize()
        te = (time.perf_counter() - t0) / args.steps
        tt = torch.tensor([te], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": F_tot / float(tt.item()) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": float(tt.item()) * 1e3,
               "note": "every step uploads the host operand pool (packed and page-locked "
                       "once at setup, like the reference's assembly) and downloads every "
                       "output block into the HMatrix"}
        del Ce
        roofline["whole_product"]["frac_e2e"] = t_roof / (e2e["ms_per_step"] * 1e-3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline_leg(args, c, A, B)
        except Exception as exc:  # pragma: no cover - reported, never fatal
            cpu = {"value": None, "unit": "GFLOP/s", "cores": None, "kind": "port",
                   "sample": f"failed: {exc!r}"}
    if rank == 0:
        rep = C.report
        line = {
            "metric": "hxh_product_fp64_gflops", "value": value, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE point cloud, GPU ACA-assembled operands)",
            "config": {"workload": configs.NAMES[args.config], "compressor": args.tag,
                       "l2": f"inputs larger than L2 (operand pools {pool_gb:.2f} GB)",
                       "parallelism": f"output-subtree partition x{world}"},
            "canonical_gflop": F_tot / 1e9, "canonical_gbytes": B_tot / 1e9,
            "phases_ms": iso,
            "phases_ms_note": "one product after the timed region without chunk overlap "
                              "(CUDA events per phase); timed steps overlap chunks on two "
                              "streams",
            "max_far_rank": rep.max_far_rank, "setup_s": setup_s,
            "operand_broadcast": ({"ms": float(sum(bcast_ms)), "bytes": int(sum(bcast_bytes)),
                                   "gbs": float(sum(bcast_bytes) / max(sum(bcast_ms), 1e-9)
                                                / 1e6)} if world > 1 else None),
            "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
            "e2e": e2e, "rel_err": rel_err, "other_compressor": alt, "clocks": ck,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def cpu_baseline_leg(args, c, A, B):
    """The reference algorithm (oracle port) on the host cores on a stratified ~20 s sample
    of this workload's units (same operands as the GPU arm, same compressor), plus ~6 s
    with one BLAS thread (the reference's own parallelism is BLAS threads only)."""
    from oracle import hmat_oracle as O
    from threadpoolctl import threadpool_limits

    table = unit_table(args.config, args.tag)
    if table is None:
        return {"value": None, "unit": "GFLOP/s", "cores": None, "kind": "port",
                "sample": f"no unit table for cfg{args.config}/{args.tag}"}
    obt = O.BlockTreeO(O.ClusterTreeO(O.make_points(c), c["n_min"]), c["eta"])
    oa = O.HMatO(obt, oracle_operand(A))
    ob = oa if B is A else O.HMatO(obt, oracle_operand(B))
    run = cpu_run(oa, ob, c["tol"], args.tag)
    s = UnitSampler(table, obt.kind, seed=1)
    s.step(run, 2.0, record=False)  # warm-up
    s.step(run, 20.0)
    v, T = s.estimate()
    out = {"value": v, "unit": "GFLOP/s", "cores": blas_threads(), "kind": "port",
           "cpu": cpu_model(), "host_cpus": os.cpu_count(), "product_s_estimate": T,
           "sample": f"reference algorithm (oracle NumPy port of hmult_new, {args.tag}) on "
                     f"{s.describe()}"}
    s1 = UnitSampler(table, obt.kind, seed=2)
    with threadpool_limits(limits=1):
        s1.step(run, 6.0)
    v1, T1 = s1.estimate()
    out["one_thread"] = {"value": v1, "unit": "GFLOP/s", "cores": 1, "product_s_estimate": T1,
                         "sample": s1.describe()}
    return out


if __name__ == "__main__":
    sys.exit(main())

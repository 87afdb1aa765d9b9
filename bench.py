"""Benchmark of the tolerance-controlled H x H product (BASELINE.json metric).

One step = one full product C = A*B on the bench workload (default: BASELINE config 2,
n=32768 on S^2, Gaussian kernel, leaf 64, eta 0.8, ACA 1e-8 operands, tol 1e-6), operands
resident in HBM: host-side term-list planning + all device phases, bracketed by CUDA
events on the product stream (barrier + synchronize on both sides; max over ranks).

value  = canonical FP64 work of the product (SURVEY 8(d) min-route model) / step time,
         in GFLOP/s, whole job.
e2e    = the same through the public API with host operands: pack/H2D of the operand pool,
         the product, D2H of every output block and construction of the HMatrix.
Multi-GPU (torchrun): output subtrees are LPT-partitioned over ranks by estimated cost,
operand pools replicated from rank 0 by an NCCL broadcast; no reduction (strong scaling).

--impl reference: the reference algorithm (the NumPy restatement in oracle/, the
reference is pure Python and cannot travel to the GPU box) on the host cores, one bounded
sample of the same workload per step.
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
def canonical_work(info, leaves, ranks):
    """F and B of the product given plan info/leaves and far ranks."""
    F = info.flops_form + info.flops_near
    B = info.bytes_form + info.bytes_near
    far = leaves["kind"] == 1
    m = leaves["m"][far].astype(float)
    n = leaves["n"][far].astype(float)
    K = leaves["K"][far].astype(float)
    fdd = leaves["fdd"][far]
    edd = leaves["edd"][far]
    r = ranks[far].astype(float)
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
    F += float(fs[pick, cols].sum())
    B += float(bs[pick, cols].sum())
    return F, B


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
    m = leaves["m"].astype(float)
    n = leaves["n"].astype(float)
    K = leaves["K"].astype(float)
    return 2 * m * n * K + leaves["fdd"] + np.where(leaves["kind"] == 1, 60 * m * n, 0.0)


# ------------------------------------------------------------------ CPU reference sample
def cpu_sample(cfg_id, c, A, budget_s, tag="aca"):
    """Reference algorithm (oracle port) on the first output leaves in DFS order until the
    time budget is spent; returns (gflop, seconds, leaves, threads)."""
    from oracle import hmat_oracle as O
    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200 import _lib, configs, hmatrix, multiply

    pts = configs.make_points(c)
    obt = O.BlockTreeO(O.ClusterTreeO(pts, c["n_min"]), c["eta"])
    _, d = multiply._host_directory(A)
    data = {}
    for b, p in A.data.items():
        data[b] = O.LR(np.ascontiguousarray(p.left), np.ascontiguousarray(p.right)) \
            if hasattr(p, "left") else np.ascontiguousarray(p)
    oa = O.HMatO(obt, data)
    leaves = [b for b in range(obt.n_nodes) if obt.kind[b] != O.INNER]
    # grow the sample geometrically until one run takes a good part of the budget
    count = 64
    t = 0.0
    while True:
        only = set(leaves[:count])
        t0 = time.perf_counter()
        Cr = O.hmult_new_o(oa, oa, O.Eps(c["tol"]), tag, only=only)
        t = time.perf_counter() - t0
        if t > 0.3 * budget_s or count >= len(leaves):
            break
        count = min(len(leaves), int(count * max(2.0, 0.5 * budget_s / max(t, 1e-3))))
    mask = np.zeros(obt.n_nodes, np.uint8)
    mask[list(only)] = 1
    plan = _lib.Plan(hmatrix.tree_arrays(A.bct), d, d, mask, multiply.plan_tile(A.bct))
    lv = plan.leaves()
    ranks = np.array([Cr.data[int(b)].rank if lv["kind"][i] == 1 else -1
                      for i, b in enumerate(lv["ids"])])
    F, _ = canonical_work(plan.info, lv, ranks)
    threads = int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))
    return F / 1e9, t, len(only), threads


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--tag", default="dense-svd")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return bench_reference(args, rank, world)
    return bench_ours(args, rank, world, local)


def bench_reference(args, rank, world):
    if rank != 0:
        return 0
    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200 import configs

    c = configs.CONFIGS[args.config]
    # operands: the same GPU-assembled A (assembly is not part of the timed product)
    bct, A, B = configs.build_operands(c)
    vals = []
    for i in range(args.warmup + args.steps):
        gf, t, nl, threads = cpu_sample(args.config, c, A, args.cpu_budget / 2, tag="aca")
        if i >= args.warmup:
            vals.append(gf / t)
    v = float(np.median(vals))
    line = {
        "impl": "reference", "metric": "hxh_product_fp64_gflops", "value": v,
        "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE point cloud)",
        "config": {"workload": configs.NAMES[args.config], "compressor": "aca"},
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": threads, "kind": "port",
                         "sample": f"reference algorithm (oracle port, NumPy/OpenBLAS) on the "
                                   f"first {nl} output leaves in DFS order per step"},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def bench_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_1805_08998_b200 as hx
    from paper_1805_08998_b200 import _lib, configs, hmatrix, multiply

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = configs.CONFIGS[args.config]
    cfg = hx.MultiplyConfig(compressor=hx.CompressorKind(args.tag), policy=hx.EpsRank(c["tol"]))
    pts = configs.make_points(c)
    bct = hx.build_block_cluster_tree(hx.build_cluster_tree(pts, c["n_min"]), c["eta"])
    h = c["n"] ** (-1.0 / 3.0)
    keep = []
    bcast_ms, bcast_bytes = [], []  # NCCL operand broadcasts (setup, outside the timed step)

    def operand(kern):
        if world == 1:
            return hx.assemble_hmatrix(kern, bct, hx.EpsRank(c["eps_a"]), pts, h=h, device=local)
        # rank 0 assembles, NCCL broadcast of the packed pool + host directory
        if rank == 0:
            H = hx.assemble_hmatrix(kern, bct, hx.EpsRank(c["eps_a"]), pts, h=h, device=local)
            n_el = H._hx_device[2]
            meta = [n_el, H._hx_packed[1], sorted(H.degraded)]
        else:
            meta = [None, None, None]
        dist.broadcast_object_list(meta, src=0)
        n_el, d, deg = meta
        buf = torch.empty(max(n_el, 1), dtype=torch.float64, device="cuda")
        if rank == 0:
            _copy_pool(H, buf, n_el)
        e0b = torch.cuda.Event(enable_timing=True)
        e1b = torch.cuda.Event(enable_timing=True)
        e0b.record()
        dist.broadcast(buf, src=0)
        e1b.record()
        torch.cuda.synchronize()
        bcast_ms.append(e0b.elapsed_time(e1b))
        bcast_bytes.append(8 * max(n_el, 1))
        keep.append(buf)
        if rank != 0:
            H = hx.HMatrix(bct, {}, set(deg))
            from paper_1805_08998_b200.assembly import _LazyLeaves
            H.data = _LazyLeaves(H)
            H._hx_packed = (None, d)
            H._hx_device = (local, buf.data_ptr(), n_el)

            class _P:  # host download path for the lazy dict / e2e leg
                def download(self_inner):
                    return buf[:n_el].cpu().numpy()
            H._hx_pool = _P()
        return H

    t_setup = time.time()
    A = operand(c["ka"])
    B = A if c["kb"] is None else operand(c["kb"])
    # partition of the output leaves (full plan once for the costs)
    _, dA = multiply.operand_directory(A)
    _, dB = multiply.operand_directory(B)
    mask = None
    if world > 1:
        full = _lib.Plan(hmatrix.tree_arrays(bct), dA, dA if B is A else dB, None,
                         multiply.plan_tile(bct))
        lv = full.leaves()
        cost = np.zeros(bct.n_nodes)
        cost[lv["ids"]] = leaf_costs(lv)
        mask = multiply.subtree_partition(
            bct, cost, world, unit_cost=lambda us: multiply.plan_unit_costs(A, B, us))[3][rank]
        full.close()
    setup_s = time.time() - t_setup
    # tensor-core work of this rank's plan (outside the timed region)
    mma = np.zeros(6)
    wp = _lib.Plan(hmatrix.tree_arrays(bct), dA, dA if B is A else dB, mask,
                   multiply.plan_tile(bct), flags=multiply.implicit_flags())
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
    F_local, B_local = canonical_work(C.plan_info, lv, C.leaf_rank)
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
        F_tot, B_tot = canonical_work(full.info, lv_all, ranks_all)
    else:
        F_tot, B_tot = F_local, B_local
    value = F_tot / (ms_max * 1e-3) / 1e9

    # e2e through the public API with host operands
    e2e = None
    if not args.no_e2e:
        pa, _ = multiply._host_directory(A)
        pb = pa if B is A else multiply._host_directory(B)[0]
        h2d = 8 * (pa.size + (0 if B is A else pb.size))
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
               "ms_per_step": float(tt.item()) * 1e3}

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
                "kernel": "grouped_gemm_kernel<Gemm64> materialization launch",
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
    # roofline time of the whole product (phase-wise max(F/P, B/BW))
    cpu = None
    if rank == 0 and world == 1 and args.cpu_budget > 0:
        try:
            gf, tcpu, nl, threads = cpu_sample(args.config, c, A, args.cpu_budget, tag="aca")
            cpu = {"value": gf / tcpu, "unit": "GFLOP/s", "cores": threads, "kind": "port",
                   "sample": f"reference algorithm (oracle NumPy port, aca compressor) on the "
                             f"first {nl} output leaves in DFS order, {tcpu:.1f}s"}
            # the reference's own parallelism is BLAS threads only: also one thread
            from threadpoolctl import threadpool_limits
            with threadpool_limits(limits=1):
                gf1, t1, nl1, _ = cpu_sample(args.config, c, A, args.cpu_budget / 4, tag="aca")
            cpu["one_thread"] = {"value": gf1 / t1, "unit": "GFLOP/s", "cores": 1,
                                 "sample": f"first {nl1} output leaves, {t1:.1f}s"}
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
                       "l2": "inputs larger than L2 (operand pools "
                             f"{8 * A._hx_device[2] / 1e9:.2f} GB)",
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
            "e2e": e2e, "clocks": ck,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _copy_pool(H, buf, n_el):
    """Device-to-device copy of a library-owned pool into a torch tensor (NCCL source)."""
    import ctypes as C

    from paper_1805_08998_b200 import _lib

    _lib.check(_lib.lib().hx_pool_download(H._hx_pool.dev.h, C.c_void_p(H._hx_pool.ptr),
                                           C.cast(C.c_void_p(buf.data_ptr()), _lib.f64p),
                                           n_el), "hx_pool_download")


if __name__ == "__main__":
    sys.exit(main())

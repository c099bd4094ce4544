#!/usr/bin/env python
"""H-LU benchmark on B200 (BASELINE.json metric, config c2 by default).

One step = R (default 16) independent accumulator H-LU factorizations of the
config-2 matrix (2D 128x128 grid, exp kernel ell=0.2, eta=2, eps=1e-6,
leaf 64; n=16384) executed in ONE persistent-scheduler launch over the
replicated lowered program; the latency of a single factorization (R=1) is
measured first and reported as ``factor_time_s``.
Inputs are resident in HBM; A is restored from a pristine copy and L2 is
flushed (256 MiB write) before every timed step, both outside the CUDA-
event bracket of the factorization.  ``value`` = algorithmic fp64 GFLOP/s
(SURVEY.md §8d formulas, counted on the device over the executed op
trace) = flops per factorization / mean factorization time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2]
  python bench.py --impl reference ...   (CPU reference arm: the oracle
                                          port of hmatdag's hlu_accu)

Under torchrun (N>1) every rank factors its own replica (config 2 is one
matrix and does not shard; replicas only, weak scaling); time is the max
over ranks of the device time.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "H-LU factor time (s) and fp64 leaf GFLOP/s vs roofline at 1/2/4/8 B200"
WORKLOADS = {
    "c4": "c4: 256 independent 1D HODLR instances, n=4096 each, exp kernel ell~U[0.05,0.5], eps=1e-6, "
          "leaf 64, standard H-LU, instances sharded across GPUs",
    "c2": "c2: 2D grid 128x128, exp kernel ell=0.2, eta=2, eps=1e-6, leaf 64, n=16384, accumulator H-LU",
    "c1": "c1: 1D HODLR n=2048, exp kernel ell=0.1, eps=1e-6, leaf 64, standard H-LU",
    "c3": "c3: 65536 points on the unit sphere, exp kernel ell=0.3, eta=2, eps=1e-5, leaf 64, "
          "accumulator H-LU",
    "c5_d3": "c5_d3: depth-3 diagonal sub-problem of c5 (n=32768 of 262144 points in the unit cube), "
             "exp kernel ell=0.25, eta=2, eps=1e-4, leaf 128, accumulator H-LU",
}


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


def fp64_peaks(torch):
    """Measured FP64 denominators on this GPU: DFMA pipe probe and cuBLAS DGEMM."""
    from paper_1911_07531_b200 import _lib

    dev = torch.cuda.current_device()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    blocks, iters = sms * 8, 20000
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(_lib.lib().hmx_fp64_fma_probe(blocks, iters, _lib.ptr(out), _lib.stream_ptr()))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = max(best, 2.0 * 8 * iters * 256 * blocks / (ms * 1e-3) / 1e12)
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    dg = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        dg = max(dg, 2.0 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    del a, b
    return {"dfma_tflops": best, "dgemm_tflops": dg}


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_profile_traffic(workload):
    """dram bytes per launch of the dominant kernel from a committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(workload)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# setup shared by both arms
# ---------------------------------------------------------------------------

def build_case(name, rank_cap):
    import torch

    from paper_1911_07531_b200 import configs, hmatrix as H

    cfg = configs.config(name)
    t0 = time.time()
    geom, root, perm, broot = configs.structure(cfg)
    pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
    t1 = time.time()
    A0 = H.assemble(broot, configs.kernel(cfg, perm), pol, rank_cap=rank_cap)
    torch.cuda.synchronize()
    t2 = time.time()
    return cfg, broot, pol, A0, {"structure_s": t1 - t0, "assembly_s": t2 - t1}


def oracle_sample(cfg, A_leaves, depth):
    """Oracle-side block tree + the sample root (diagonal block at `depth`)."""
    from oracle import hm_oracle as O

    ct = O.cluster_tree(cfg.points, cfg.n_min)
    adm = O.adm_weak(ct) if cfg.admissibility == "weak" else O.adm_standard(ct, cfg.eta)
    bt = O.block_tree(ct, adm)
    u = 0
    for _ in range(depth):
        if bt.leaf(u):
            break
        u = bt.kids[u][0]
    lv = {v: A_leaves[v] for v in bt.leaves(u)}
    return O, bt, u, lv


_JOB = None


def _oracle_job(_i):
    """Pool worker: one sample factorization of the forked-in job."""
    return _oracle_run(_JOB)


def _oracle_run(args):
    O, bt, u, lv, mode, pol = args
    from threadpoolctl import threadpool_limits

    A = O.HM(bt, {k: (x[0], *[y.copy() for y in x[1:]]) for k, x in lv.items()})
    L, U = O.HM(bt, {}), O.HM(bt, {})
    for v in lv:
        m, n = bt.shape(v)
        for M in (L, U):
            M.lv[v] = ("R", np.zeros((m, 0)), np.zeros((n, 0))) if bt.adm[v] else ("D", np.zeros((m, n)))
    O.COUNT.flops = 0.0
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        if mode == "std":
            O.hlu(A, L, U, u, pol)
        else:
            O.hlu_accu(A, L, U, u, O.Accs(), pol)
        dt = time.perf_counter() - t0
    return dt, O.COUNT.flops


SAMPLE_DEPTH = {"c2": 1, "c1": 0, "c4_0": 0}


def cpu_baseline(cfg, A_leaves, reps=2):
    """Oracle port on this host, 1 thread, on a bounded sample (10-30 s)."""
    depth = SAMPLE_DEPTH.get(cfg.name, 1)
    O, bt, u, lv = oracle_sample(cfg, A_leaves, depth)
    pol = O.Policy("accuracy", eps=cfg.eps)
    tot_t, tot_f = 0.0, 0.0
    for _ in range(reps):
        dt, fl = _oracle_run((O, bt, u, lv, cfg.mode, pol))
        tot_t += dt
        tot_f += fl
    return {"value": tot_f / tot_t / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "port",
            "sample": f"{'hlu_accu' if cfg.mode == 'accu' else 'hlu'} of the depth-{depth} "
                      f"diagonal block ({bt.shape(u)[0]}x{bt.shape(u)[1]}) of {cfg.name}, "
                      f"{reps} reps, 1 BLAS thread, oracle/hm_oracle.py",
            "seconds": tot_t}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import multiprocessing as mp

    import torch

    cfg, broot, pol, A0, setup = build_case(args.config, args.rank_cap)
    A_leaves = A0.store.download_leaves()
    del A0
    torch.cuda.empty_cache()
    depth = SAMPLE_DEPTH.get(cfg.name, 1)
    O, bt, u, lv = oracle_sample(cfg, A_leaves, depth)
    opol = O.Policy("accuracy", eps=cfg.eps)
    ncores = len(os.sched_getaffinity(0))
    nproc = max(1, min(ncores, 32))
    global _JOB
    _JOB = (O, bt, u, lv, cfg.mode, opol)
    ctx = mp.get_context("fork")
    with ctx.Pool(nproc) as pool:
        for _ in range(args.warmup):
            pool.map(_oracle_job, range(nproc))
        t0 = time.perf_counter()
        flops = 0.0
        for _ in range(args.steps):
            res = pool.map(_oracle_job, range(nproc))
            flops += sum(r[1] for r in res)
        wall = time.perf_counter() - t0
    value = flops / wall / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS.get(cfg.name, cfg.name),
                   "sample": f"{nproc} concurrent oracle {('hlu_accu' if cfg.mode == 'accu' else 'hlu')}"
                             f" factorizations of the depth-{depth} diagonal block "
                             f"({bt.shape(u)[0]}x{bt.shape(u)[1]}) per step"},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": nproc, "kind": "port",
                         "sample": f"oracle/hm_oracle.py (numpy/scipy restatement of hmatdag), "
                                   f"{nproc} processes x 1 BLAS thread, depth-{depth} diagonal "
                                   f"block of {cfg.name}; input H-matrix assembled on the GPU "
                                   f"(setup, untimed)"},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hmx", choices=["hmx", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--exec", default="persistent", choices=["persistent", "graph", "wave"])
    ap.add_argument("--rank-cap", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--instances", type=int, default=256, help="config 4 batch size (total)")
    ap.add_argument("--ctas-per-sm", type=int, default=0,
                    help="executor variant for the batched run (0 = auto: 2 when replicas > 1)")
    ap.add_argument("--replicas", type=int, default=16,
                    help="independent factorizations per GPU per step (throughput)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "c4":
        return run_c4(args)

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    from paper_1911_07531_b200 import engine, hmatrix as H
    from paper_1911_07531_b200.arith import get_plan

    cfg, broot, pol, A0, setup = build_case(args.config, args.rank_cap)
    em = {"persistent": engine.EXEC_PERSISTENT, "graph": engine.EXEC_GRAPH,
          "wave": engine.EXEC_WAVE}[args.exec]
    flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
    R = max(1, args.replicas)

    def timed_run(plan, Ast, A0st, Lst, Ust, steps, warmup, sampler=None):
        def one():
            Ast.copy_from(A0st)
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.run(Ast, Lst, Ust, em, check=False)
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1)

        for _ in range(warmup):
            one()
        plan.check()
        barrier()
        torch.cuda.synchronize()
        if sampler is not None:
            with sampler:
                ms = [one() for _ in range(steps)]
        else:
            ms = [one() for _ in range(steps)]
        barrier()
        plan.check()
        return float(np.mean(ms))

    def max_over_ranks(x):
        if dist is None:
            return x
        tt = torch.tensor([x], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    # 1) latency of ONE factorization (the BASELINE factor time)
    t0 = time.time()
    plan1 = get_plan(A0.table, cfg.mode, pol, args.rank_cap)
    setup["plan_s"] = time.time() - t0
    A1 = A0.copy()
    L1, U1 = H.zeros(broot, pol, args.rank_cap), H.zeros(broot, pol, args.rank_cap)
    t_single = max_over_ranks(timed_run(plan1, A1.store, A0.store, L1.store, U1.store,
                                        args.steps, args.warmup))
    c = plan1.counters()
    flops = float(c["flops"])
    alg_bytes = float(c["bytes"])

    # 2) throughput: R independent factorizations per GPU in one launch (the
    #    single-matrix critical path leaves most SMs idle; a batch fills them)
    clk = ClockSampler(local)
    if R > 1:
        del A1, L1, U1
        t0 = time.time()
        planR = get_plan(A0.table, cfg.mode, pol, args.rank_cap, nrep=R,
                         ctas_per_sm=args.ctas_per_sm or None)
        setup["plan_batch_s"] = time.time() - t0
        AB0 = H.HBatch.replicate(A0, R)
        AB = H.HBatch(broot, pol, R, args.rank_cap)
        LB, UB = H.HBatch(broot, pol, R, args.rank_cap), H.HBatch(broot, pol, R, args.rank_cap)
        t_step = max_over_ranks(timed_run(planR, AB.store, AB0.store, LB.store, UB.store,
                                          args.steps, args.warmup, clk))
        planT = planR
    else:
        AB0 = AB = LB = UB = None
        A1 = A0.copy()
        L1, U1 = H.zeros(broot, pol, args.rank_cap), H.zeros(broot, pol, args.rank_cap)
        t_step = max_over_ranks(timed_run(plan1, A1.store, A0.store, L1.store, U1.store,
                                          args.steps, 0, clk))
        planT = plan1
    value = world * R * flops / (t_step * 1e-3) / 1e9

    # end to end through the public API with host buffers (pinned), the same
    # batch: H2D of every A, factorization, D2H of every L and U
    e2e = None
    if not args.no_e2e:
        from paper_1911_07531_b200.arith import hlu_batch

        if R == 1:
            AB0 = H.HBatch.replicate(A0, 1)
            AB = H.HBatch(broot, pol, 1, args.rank_cap)
            LB, UB = H.HBatch(broot, pol, 1, args.rank_cap), H.HBatch(broot, pol, 1, args.rank_cap)
        # the caller's A in host memory, packed (live leaf data at the actual
        # ranks, hmatrix.pack_leaves format) in pinned buffers
        hA_v, hA_r = AB0.download_packed()
        torch.cuda.synchronize()
        hA_v, hA_r = hA_v.clone().pin_memory(), hA_r.clone().pin_memory()
        # pipelined host -> device -> host stream of batches (batch.PipelinedHLU):
        # the H2D of batch i+1 and the D2H of batch i-1 overlap the
        # factorization of batch i; every batch moves its own packed A in and
        # its packed L, U (+ rank words) out, all inside the timed region
        from paper_1911_07531_b200.batch import PipelinedHLU

        del AB, LB, UB
        torch.cuda.empty_cache()
        pipe = PipelinedHLU(broot, pol, R, args.rank_cap, cfg.mode, em)
        inputs = [(hA_v, hA_r)] * max(2, args.warmup)
        res, ev = pipe.run(inputs)
        torch.cuda.synchronize()
        pipe.check()
        outs = [res[0], res[1]]
        K = args.steps
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(pipe.s_h2d)
        res, ev = pipe.run([(hA_v, hA_r)] * K, [outs[i & 1] for i in range(K)])
        e1.record(pipe.s_d2h)
        torch.cuda.synchronize()
        pipe.check()
        te = max_over_ranks(e0.elapsed_time(e1) / K)
        (hL, hLr), (hU, hUr) = res[-1]
        d2h = (hL.numel() + hU.numel()) * 8 + (hLr.numel() + hUr.numel()) * 4
        vb = hA_v.numel() * 8 + hA_r.numel() * 4
        e2e = {"value": world * R * flops / (te * 1e-3) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(vb), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": te, "api": "batch.PipelinedHLU: per step H2D of the packed A batch, unpack, hlu_batch plan, pack, D2H of packed L and U (pinned host buffers); steps pipelined on h2d / compute / d2h streams, K steps in one bracket"}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0

    peaks = fp64_peaks(torch)
    hbm, hbm_src = hbm_peak()
    achieved = R * flops / (t_step * 1e-3) / 1e12
    traffic = load_profile_traffic(cfg.name)
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peaks["dgemm_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["dgemm_tflops"],
                "traffic": traffic,
                "peak_source": "FP64 DMMA: torch/cuBLAS DGEMM 8192^3 measured in this run "
                               "(MEASURED_PEAKS.json has no FP64 entry)",
                "dfma_peak_tflops": peaks["dfma_tflops"],
                "algorithmic_bytes_per_step": R * alg_bytes,
                "hbm_achieved_gbs": R * alg_bytes / (t_step * 1e-3) / 1e9,
                "hbm_peak_gbs": hbm, "hbm_peak_source": hbm_src,
                "kernel": f"k_persistent (one launch per step = {R} factorizations)"}
    cpub = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpub = cpu_baseline(cfg, A0.store.download_leaves())
        except Exception as e:  # reported, never fatal for the GPU number
            cpub = {"error": repr(e)}
    stats = plan1.stats()
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS.get(cfg.name, cfg.name), "n": int(cfg.n),
                   "mode": cfg.mode, "dag": plan1.dag_mode, "executor": args.exec,
                   "rank_cap": args.rank_cap,
                   "replicas_per_gpu": R, "ctas_per_sm": planT.ctas_per_sm,
                   "step": f"{R} independent factorizations of the config matrix per GPU "
                           "in one launch (replicated plan)",
                   "parallelism": f"replicas x{world}",
                   "l2": "flushed by a 256 MiB write before every timed step",
                   "tasks": stats["tasks"], "ops": stats["ops"], "waves": stats["waves"]},
        "factor_time_s": t_single * 1e-3,
        "factor_time_note": "latency of ONE factorization (R=1 plan), max over ranks",
        "gflop_per_factorization": flops / 1e9,
        "truncations": c["truncations"],
        "roofline": roofline,
        "cpu_baseline": cpub,
        "e2e": e2e,
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
        "setup": setup,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def run_c4(args):
    """Config 4: 256 instances sharded over ranks, one batched plan per rank
    (strong scaling: the total batch is fixed)."""
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1911_07531_b200 import engine
    from paper_1911_07531_b200.batch import InstanceBatch, shard

    ids = list(shard(args.instances, world, rank))
    t0 = time.time()
    batch = InstanceBatch(ids, rank_cap=args.rank_cap)
    setup_s = time.time() - t0
    flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")

    def step():
        batch.A.copy_from(batch.A0)
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        batch.plan.run(batch.A, batch.L, batch.U, engine.EXEC_PERSISTENT, check=False)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for _ in range(args.warmup):
        step()
    batch.plan.check()
    flops = float(batch.plan.counters()["flops"])
    if dist is not None:
        dist.barrier()
    ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            ms.append(step())
    t = float(np.mean(ms))
    tot = torch.tensor([t, flops], dtype=torch.float64, device="cuda")
    if dist is not None:
        tmax = tot[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        fl = tot[1:].clone()
        dist.all_reduce(fl, op=dist.ReduceOp.SUM)
        t, flops_all = float(tmax.item()), float(fl.item())
    else:
        flops_all = flops
    if rank == 0:
        peaks = fp64_peaks(torch)
        ach = flops / (float(np.mean(ms)) * 1e-3) / 1e12
        line = {"metric": METRIC, "value": flops_all / (t * 1e-3) / 1e9, "unit": "GFLOP/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": WORKLOADS["c4"], "instances": args.instances,
                           "instances_per_gpu": len(ids), "rank_cap": args.rank_cap,
                           "parallelism": f"instances sharded x{world}",
                           "l2": "flushed by a 256 MiB write before every timed step"},
                "roofline": {"bound": "tensor", "achieved": ach, "peak": peaks["dgemm_tflops"],
                             "unit": "TFLOP/s", "frac": ach / peaks["dgemm_tflops"],
                             "traffic": load_profile_traffic("c4"),
                             "peak_source": "FP64 DMMA: torch/cuBLAS DGEMM measured in this run"},
                "gpu_launches": args.steps, "clocks": clk.summary(),
                "setup": {"assembly_and_plan_s": setup_s}}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""H-LU benchmark on B200 (BASELINE.json metric; config c3 by default).

A step is ONE H-LU factorization of the named config's matrix (default c3:
65536 points on the unit sphere, exp kernel ell=0.3, eta=2, eps=1e-5,
leaf 64, accumulator H-LU — the largest BASELINE config one GPU factors;
c5 is selected with --config c5).  The factorization is one
persistent-scheduler launch (k_persistent, 1 CTA per SM) over the lowered
task DAG.  Inputs are resident in HBM (the A pool is larger than L2) and A
is restored from a pristine device copy before every step, outside the
CUDA-event bracket.  ``value`` = algorithmic fp64 GFLOP/s (SURVEY.md §8d
formulas, counted on the device over the executed op trace) = flops of one
factorization / its mean time; ``factor_time_s`` = that time.

After the timed steps the factors of the last step are checked against the
reference's own run (tests/golden/<cfg>.npz, tests/golden/<cfg>_leaves.npz):
every L/U block rank, per-block Frobenius norms and the entries of sampled
leaves.  A failed check prints ``value: null`` with the reason.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1|c2|c3|c4|c5|c5_d3]
  python bench.py --impl reference ...  (the reference's CPU path, restated
                                         in oracle/hm_oracle.py, on the same
                                         config, assembled on the CPU)

Under torchrun (N>1): the single-matrix configs run ONE factorization
partitioned over the ranks by block rows (run_partitioned: strong scaling,
partition.DistributedHLU); c4 shards its 256 instances over the ranks (no
collective on the data path).  HMX_BENCH_REPLICAS=1: one independent
factorization per rank instead.  Time is the max over ranks of the device
time.
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
    "c1": "c1: 1D HODLR n=2048, exp kernel ell=0.1, eps=1e-6, leaf 64, standard H-LU",
    "c2": "c2: 2D grid 128x128, exp kernel ell=0.2, eta=2, eps=1e-6, leaf 64, n=16384, accumulator H-LU",
    "c3": "c3: 65536 points on the unit sphere, exp kernel ell=0.3, eta=2, eps=1e-5, leaf 64, "
          "accumulator H-LU",
    "c4": "c4: 256 independent 1D HODLR instances, n=4096 each, exp kernel ell~U[0.05,0.5], eps=1e-6, "
          "leaf 64, standard H-LU, instances sharded across GPUs",
    "c5": "c5: 262144 points uniform in the unit cube, exp kernel ell=0.25, eta=2, eps=1e-4, leaf 128, "
          "accumulator H-LU",
    "c5_d3": "c5_d3: depth-3 diagonal sub-problem of c5 (n=32768 of 262144 points in the unit cube), "
             "exp kernel ell=0.25, eta=2, eps=1e-4, leaf 128, accumulator H-LU",
}
RANK_CAP = {"c5": 128, "c5_d3": 128}
# cpu_baseline sample of the GPU arm: the diagonal block at this depth (10-30 s of oracle work)
SAMPLE_DEPTH = {"c1": 0, "c2": 1, "c3": 2, "c5_d3": 2, "c5": 4}


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


def rank_cap_of(name, arg):
    return arg if arg else RANK_CAP.get(name, 64)


# ---------------------------------------------------------------------------
# parity of the timed factors vs the reference's own run
# ---------------------------------------------------------------------------

def parity_report(cfg, mode, L, U):
    from tests import parity as PT
    from tests.golden_inputs import have, load

    out = {"fixture": None}
    if not have(cfg.name):
        out["note"] = "no reference fixture for this config (c5: numerics beyond the CPU reference)"
        return out, True
    meta, arr = load(cfg.name)
    if f"{mode}_L_rank" not in arr:
        out["note"] = f"fixture has no {mode} run"
        return out, True
    out["fixture"] = f"tests/golden/{cfg.name}.npz ({mode})"
    Lr, Ur = L.store.ranks.cpu().numpy(), U.store.ranks.cpu().numpy()
    out["rank_mismatches"] = PT.compare_ranks(arr, mode, Lr, Ur)
    lay = L.store.layout
    rel, ab = [], []
    for which, M in (("L", L), ("U", U)):
        f = PT.store_fro(lay, M.store.values.cpu().numpy(), M.store.ranks.cpu().numpy())
        r_, a_ = PT.compare_fro(arr, mode, which, f)
        rel.append(r_)
        ab.append(a_)
    out["block_fro_max_rel"] = max(rel)
    out["block_fro_max_abs_over_factor"] = max(ab)
    samples = PT.leaf_samples(cfg.name)
    if samples is not None:
        stores = {"L": L.store, "U": U.store}
        totals = {w: PT.factor_norm(arr, mode, w) for w in ("L", "U")}
        worst, nblk = PT.compare_leaf_samples(samples, mode, lambda w, u: stores[w].download_leaf(u),
                                              totals)
        out["leaf_entries_max_rel"] = worst
        out["leaf_blocks_compared"] = nblk
    tol = 10 * cfg.eps
    out["tolerance"] = (f"ranks equal; per-block Frobenius difference relative to the block (blocks with "
                        f">= {PT.SIGNIFICANT:g} of the factor norm) and to the factor norm (all blocks), "
                        f"sampled leaf entries relative to max(block, {PT.SIGNIFICANT:g} x factor): "
                        f"all <= 10*eps = {tol:g}")
    ok = (out["rank_mismatches"] == 0 and out["block_fro_max_rel"] <= tol
          and out["block_fro_max_abs_over_factor"] <= tol
          and out.get("leaf_entries_max_rel", 0.0) <= tol)
    out["ok"] = bool(ok)
    return out, ok


# ---------------------------------------------------------------------------
# CPU reference arm (no GPU, no product library)
# ---------------------------------------------------------------------------

_JOB = None


def _assemble_chunk(leaves):
    O, bt, fn, pol = _JOB
    return O.assemble_leaves(bt, fn, pol, leaves)


def cpu_structure_and_matrix(cfg, nproc):
    """Oracle block tree and A assembled on the host (kernel evaluation;
    dense_to_lowrank for admissible blocks <= 128, randomized range finder
    above: oracle.assemble_leaves), leaves split over ``nproc`` processes."""
    import multiprocessing as mp

    from threadpoolctl import threadpool_limits

    from oracle import hm_oracle as O

    ct = O.cluster_tree(cfg.points, cfg.n_min)
    adm = O.adm_weak(ct) if cfg.admissibility == "weak" else O.adm_standard(ct, cfg.eta)
    bt = O.block_tree(ct, adm)
    pol = O.Policy("accuracy", eps=cfg.eps)
    fn = (lambda pts, perm, ell: (lambda I, J: O.exp_kernel_dense(pts, perm, ell, I, J)))(
        cfg.points, ct.perm, cfg.ell)
    leaves = bt.leaves(0)
    global _JOB
    _JOB = (O, bt, fn, pol)
    chunks = [leaves[i::nproc * 4] for i in range(nproc * 4)]
    lv = {}
    with threadpool_limits(limits=1):
        if nproc > 1:
            with mp.get_context("fork").Pool(nproc) as pool:
                for part in pool.map(_assemble_chunk, chunks):
                    lv.update(part)
        else:
            lv = O.assemble_leaves(bt, fn, pol, leaves)
    return O, bt, O.HM(bt, lv), pol


def _oracle_factor(O, A, u, mode, pol):
    """One oracle factorization of the block u of A (1 BLAS thread);
    returns (seconds, algorithmic flops, truncations)."""
    from threadpoolctl import threadpool_limits

    W = A.copy()
    L, U = O.zeros(A.bt), O.zeros(A.bt)
    O.COUNT.flops = 0.0
    O.COUNT.truncations = O.COUNT.updates = 0
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        if mode == "std":
            O.hlu(W, L, U, u, pol)
        else:
            O.hlu_accu(W, L, U, u, O.Accs(), pol)
        dt = time.perf_counter() - t0
    return dt, O.COUNT.flops, O.COUNT.truncations


def _c4_instance(j):
    from paper_1911_07531_b200 import configs

    cfg = configs.config(f"c4_{j}")
    O, bt, A, pol = cpu_structure_and_matrix(cfg, 1)
    return _oracle_factor(O, A, 0, "std", pol)


def run_reference(args):
    """The reference's CPU path on the SAME config: hmatdag's recursive
    arith.hlu / accumulator.hlu_accu as restated in oracle/hm_oracle.py
    (pinned bit-exactly to the unmodified reference, tests/test_oracle.py),
    on an H-matrix assembled on the host.  No GPU and no product library is
    touched.  c4: the 256 instances over all host cores (one process per
    core, 1 BLAS thread each); other configs: one factorization, 1 BLAS
    thread (the fastest setting for the reference), repeated
    while the budget allows."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_1911_07531_b200 import configs

    ncores = len(os.sched_getaffinity(0))
    name = args.config
    t_setup = time.time()
    if name == "c4":
        import multiprocessing as mp

        nproc = max(1, min(ncores, 64))
        ids = list(range(args.instances))
        times, flops = [], 0.0
        with mp.get_context("fork").Pool(nproc) as pool:
            for step in range(max(1, args.steps)):
                t0 = time.perf_counter()
                res = pool.map(_c4_instance, ids)
                times.append(time.perf_counter() - t0)
                flops = sum(r[1] for r in res)
                if sum(times) > args.ref_budget:
                    break
        sec = float(np.median(times))
        value = flops / sec / 1e9
        sample = (f"all {len(ids)} instances per step (host assembly + oracle hlu per instance), "
                  f"{nproc} processes x 1 BLAS thread; median of {len(times)} steps")
        cores = nproc
        steps_run = len(times)
        extra = {"instances": len(ids)}
    else:
        if name == "c5":
            print(json.dumps({"impl": "reference", "unavailable":
                              "c5 numerics are beyond the CPU reference (assembly ~8e15 flop as dense "
                              "SVDs, H-LU days; SURVEY.md §8c)"}), flush=True)
            return 0
        cfg = configs.config(name)
        mode = args.mode or cfg.mode
        O, bt, A, pol = cpu_structure_and_matrix(cfg, max(1, min(ncores, 64)))
        setup_s = time.time() - t_setup
        times, tr = [], 0
        for step in range(max(1, args.steps)):
            dt, flops, tr = _oracle_factor(O, A, 0, mode, pol)
            times.append(dt)
            if sum(times) + dt > args.ref_budget:
                break
        sec = float(np.median(times))
        value = flops / sec / 1e9
        cores = 1
        steps_run = len(times)
        sample = (f"the full {name} matrix, {'hlu_accu' if mode == 'accu' else 'hlu'} "
                  f"(oracle/hm_oracle.py restatement of hmatdag), 1 BLAS thread, median of "
                  f"{steps_run} factorization(s) (steps beyond the {args.ref_budget:.0f} s budget "
                  f"skipped); A assembled on the host ({setup_s:.0f} s, untimed)")
        extra = {"factor_time_s": sec, "truncations": int(tr), "mode": mode,
                 "gflop_per_factorization": flops / 1e9, "min_s": float(min(times)),
                 "max_s": float(max(times))}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": steps_run, "steps_requested": args.steps,
        "warmup": 0, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong" if name == "c4" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS.get(name, name), "same_config": True},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": "port",
                         "sample": sample, "ncores_host": ncores},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    line.update(extra)
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
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


def cpu_baseline(cfg, mode, A_leaves):
    """Oracle port on this host, 1 thread, on a bounded sample (the diagonal
    block at SAMPLE_DEPTH of the same matrix, 10-30 s)."""
    from oracle import hm_oracle as O

    ct = O.cluster_tree(cfg.points, cfg.n_min)
    adm = O.adm_weak(ct) if cfg.admissibility == "weak" else O.adm_standard(ct, cfg.eta)
    bt = O.block_tree(ct, adm)
    u = 0
    depth = SAMPLE_DEPTH.get(cfg.name, 1)
    for _ in range(depth):
        if bt.leaf(u):
            break
        u = bt.kids[u][0]
    A = O.HM(bt, {v: A_leaves[v] for v in bt.leaves(u)})
    pol = O.Policy("accuracy", eps=cfg.eps)
    dt, fl, _ = _oracle_factor(O, A, u, mode, pol)
    return {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "port",
            "sample": f"{'hlu_accu' if mode == 'accu' else 'hlu'} of the depth-{depth} diagonal block "
                      f"({bt.shape(u)[0]}x{bt.shape(u)[1]}) of {cfg.name}, 1 BLAS thread, "
                      f"oracle/hm_oracle.py", "seconds": dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hmx", choices=["hmx", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--mode", default=None, choices=[None, "std", "accu"])
    ap.add_argument("--exec", default="persistent", choices=["persistent", "graph", "wave"])
    ap.add_argument("--rank-cap", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--instances", type=int, default=256, help="config 4 batch size (total)")
    ap.add_argument("--replicas", type=int, default=1,
                    help="also time R independent factorizations in one launch (throughput key)")
    ap.add_argument("--ref-budget", type=float, default=240.0,
                    help="reference arm: seconds of CPU factorization before further steps are skipped")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "c4":
        return run_c4(args)
    if args.config == "c5":
        return run_c5(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1 and not os.environ.get("HMX_BENCH_REPLICAS"):
        return run_partitioned(args)
    return run_single(args)


def run_c5(args):
    """Config 5 (n = 262144) on ONE GPU: rank-first assembly with rank-bounded
    arenas, native lowering, one factorization (tools/run_c5.py).  One step
    takes minutes; the L / U ranks of the full problem exceed what one B200
    holds, so the run reports HMX_ERR_RANK_OVERFLOW and
    its probe residual measures the clipping: `value` is withheld then."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import run_c5 as R5
    import torch

    rep = R5.run("c5", log=lambda *a, **k: None)
    ok = rep.get("status", 1) == 0
    peaks = fp64_peaks(torch)
    value = rep["gflops"]
    line = {
        "metric": METRIC, "value": value if ok else None, "unit": "GFLOP/s", "n_gpus": 1, "steps": 1,
        "warmup": 0, "ms_per_step": rep["factor_s"] * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS.get("c5", "c5"), "n": 262144, "mode": "accu",
                   "step": "one H-LU factorization (one k_persistent launch)", "parallelism": "single GPU",
                   "l2": "inputs larger than L2", "plan": rep.get("plan")},
        "factor_time_s": rep["factor_s"], "gflop_per_factorization": rep["gflop"],
        "truncations": rep["truncations"], "probe_residual": rep.get("probe_residual"),
        "status": rep.get("status"), "leaves_at_cap": rep.get("leaves_at_cap"),
        "peak_mem_gb": rep.get("peak_mem_gb"),
        "roofline": {"bound": "tensor", "achieved": value / 1e3, "peak": peaks["dgemm_tflops"],
                     "unit": "TFLOP/s", "frac": value / 1e3 / peaks["dgemm_tflops"], "traffic": None,
                     "kernel": "k_persistent<1>"},
        "cpu_baseline": None, "e2e": None, "gpu_launches": 1,
        "setup": {k: rep.get(k) for k in ("structure_s", "assembly_s", "plan_s")},
    }
    if not ok:
        line["value_withheld"] = ("rank bounds that fit one GPU clip L / U blocks (status %s); "
                                  "value_unchecked is the clipped run" % rep.get("status"))
        line["value_unchecked"] = value
    print(json.dumps(line), flush=True)
    return 0


def run_partitioned(args):
    """N > 1: ONE factorization of the config matrix partitioned over the
    ranks by block rows (partition.DistributedHLU: peer-memory exchange along
    DAG edges, no collective on the data path).  Strong scaling: the total
    work is fixed.  HMX_BENCH_REPLICAS=1 restores one matrix per GPU."""
    import torch
    import torch.distributed as dist

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1911_07531_b200 import hmatrix as H
    from paper_1911_07531_b200.partition import DistributedHLU

    rc = rank_cap_of(args.config, args.rank_cap)
    cfg, broot, pol, A0, setup = build_case(args.config, rc)
    mode = args.mode or cfg.mode
    t0 = time.time()
    d = DistributedHLU(A0.table, mode, pol, rc)
    setup["plan_s"] = time.time() - t0
    A, L, U = d.stores(A0.store)
    d.connect(A, L, U)
    clk = ClockSampler(local)

    def one():
        A.copy_from(A0.store)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d.run(events=(e0, e1))
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for _ in range(args.warmup):
        one()
    dist.barrier()
    torch.cuda.synchronize()
    with clk:
        per_step = [one() for _ in range(args.steps)]
    dist.barrier()
    tt = torch.tensor([float(np.mean(per_step))], device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    c = d.pp.plan.counters()
    cc = torch.tensor([float(c[1]), float(c[2]), float(c[0])], device="cuda", dtype=torch.float64)
    dist.all_reduce(cc)
    flops, alg_bytes, ntrunc = (float(x) for x in cc.tolist())
    Lf, Uf = d.collect(L, 1), d.collect(U, 2)
    st = d.part.stats()
    d.close()
    if rank != 0:
        dist.destroy_process_group()
        return 0
    Lh, Uh = H.HMatrix(Lf, 0, pol), H.HMatrix(Uf, 0, pol)
    par, ok = ({"skipped": True}, True) if args.no_parity else parity_report(cfg, mode, Lh, Uh)
    peaks = fp64_peaks(torch)
    hbm, hbm_src = hbm_peak()
    value = flops / (t_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value if ok else None, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS.get(cfg.name, cfg.name), "n": int(cfg.n), "mode": mode,
                   "executor": "persistent (one launch per rank, ranks release each other's tasks)",
                   "rank_cap": rc,
                   "step": "one H-LU factorization of the config matrix partitioned over the ranks",
                   "parallelism": f"block-row partition x{world} (peer-memory exchange along DAG edges)",
                   "partition": st},
        "factor_time_s": t_ms * 1e-3,
        "factor_time_steps_s": [x * 1e-3 for x in per_step],
        "gflop_per_factorization": flops / 1e9,
        "truncations": int(ntrunc),
        "parity": par,
        "roofline": {"bound": "tensor", "achieved": value / 1e3, "peak": world * peaks["dgemm_tflops"],
                     "unit": "TFLOP/s", "frac": value / 1e3 / (world * peaks["dgemm_tflops"]),
                     "traffic": None,
                     "peak_source": "FP64: torch/cuBLAS DGEMM 8192^3 measured in this run, x n_gpus",
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "hbm_achieved_gbs": alg_bytes / (t_ms * 1e-3) / 1e9, "hbm_peak_gbs": world * hbm,
                     "hbm_peak_source": hbm_src,
                     "kernel": "k_persistent<1> (one launch per rank = its share of one factorization)"},
        "cpu_baseline": None,
        "e2e": None,
        "gpu_launches": args.steps * world,
        "clocks": clk.summary(),
        "setup": setup,
    }
    if not ok:
        line["value_withheld"] = "factors failed the parity check against the reference fixture"
        line["value_unchecked"] = value
    print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


def run_single(args):
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

    def max_over_ranks(x):
        if dist is None:
            return x
        tt = torch.tensor([x], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    from paper_1911_07531_b200 import engine, hmatrix as H
    from paper_1911_07531_b200.arith import get_plan

    rc = rank_cap_of(args.config, args.rank_cap)
    cfg, broot, pol, A0, setup = build_case(args.config, rc)
    mode = args.mode or cfg.mode
    em = {"persistent": engine.EXEC_PERSISTENT, "graph": engine.EXEC_GRAPH,
          "wave": engine.EXEC_WAVE}[args.exec]
    big = A0.store.values.numel() * 8 > 2 * 126 * 2**20
    flush = None if big else torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")

    def timed_run(plan, Ast, A0st, Lst, Ust, steps, warmup, sampler=None):
        def one():
            Ast.copy_from(A0st)
            if flush is not None:
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
        return float(np.mean(ms)), ms

    # ONE factorization per step (1 CTA per SM executor)
    t0 = time.time()
    plan1 = get_plan(A0.table, mode, pol, rc)
    setup["plan_s"] = time.time() - t0
    A1 = A0.copy()
    L1, U1 = H.zeros(broot, pol, rc), H.zeros(broot, pol, rc)
    clk = ClockSampler(local)
    t_ms, per_step = timed_run(plan1, A1.store, A0.store, L1.store, U1.store, args.steps,
                               args.warmup, clk)
    t_ms = max_over_ranks(t_ms)
    c = plan1.counters()
    flops = float(c["flops"])
    alg_bytes = float(c["bytes"])
    par, ok = ({"skipped": True}, True) if args.no_parity else parity_report(cfg, mode, L1, U1)
    value = world * flops / (t_ms * 1e-3) / 1e9

    batched = None
    if args.replicas > 1:
        del A1
        R = args.replicas
        planR = get_plan(A0.table, mode, pol, rc, nrep=R)
        AB0 = H.HBatch.replicate(A0, R)
        AB = H.HBatch(broot, pol, R, rc)
        LB, UB = H.HBatch(broot, pol, R, rc), H.HBatch(broot, pol, R, rc)
        tb, _ = timed_run(planR, AB.store, AB0.store, LB.store, UB.store, args.steps, args.warmup)
        tb = max_over_ranks(tb)
        batched = {"replicas_per_gpu": R, "ms_per_launch": tb, "ctas_per_sm": planR.ctas_per_sm,
                   "value": world * R * flops / (tb * 1e-3) / 1e9, "unit": "GFLOP/s",
                   "note": "R independent factorizations of the config matrix in one launch "
                           "(replicated plan); throughput only, not the headline"}
        del AB0, AB, LB, UB, planR
        torch.cuda.empty_cache()

    # end to end through the public API with host buffers: per step the H2D
    # of the packed A (pinned), unpack, factorization, pack, D2H of packed L
    # and U (batch.PipelinedHLU, steps pipelined on three streams)
    e2e = None
    if not args.no_e2e:
        from paper_1911_07531_b200.batch import PipelinedHLU

        AB0 = H.HBatch.replicate(A0, 1)
        hA_v, hA_r = AB0.download_packed()
        torch.cuda.synchronize()
        hA_v, hA_r = hA_v.clone().pin_memory(), hA_r.clone().pin_memory()
        del AB0
        torch.cuda.empty_cache()
        pipe = PipelinedHLU(broot, pol, 1, rc, mode, em)
        res, ev = pipe.run([(hA_v, hA_r)] * max(2, args.warmup))
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
        e2e = {"value": world * flops / (te * 1e-3) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(vb), "d2h_bytes_per_step": int(d2h), "ms_per_step": te,
               "api": "batch.PipelinedHLU (hlu_accu / hlu plan): per step H2D of the packed A from "
                      "pinned host memory, unpack, factorization, pack, D2H of packed L and U; "
                      "steps pipelined on h2d / compute / d2h streams, K steps in one bracket"}
        del pipe
        torch.cuda.empty_cache()

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0

    peaks = fp64_peaks(torch)
    hbm, hbm_src = hbm_peak()
    achieved = flops / (t_ms * 1e-3) / 1e12
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peaks["dgemm_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["dgemm_tflops"],
                "traffic": load_profile_traffic(f"{cfg.name}_{mode}"),
                "peak_source": "FP64: torch/cuBLAS DGEMM 8192^3 measured in this run "
                               "(MEASURED_PEAKS.json has no FP64 entry)",
                "dfma_peak_tflops": peaks["dfma_tflops"],
                "algorithmic_bytes_per_launch": alg_bytes,
                "hbm_achieved_gbs": alg_bytes / (t_ms * 1e-3) / 1e9,
                "hbm_peak_gbs": hbm, "hbm_peak_source": hbm_src,
                "kernel": "k_persistent<1> (one launch = one factorization)"}
    cpub = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpub = cpu_baseline(cfg, mode, A0.store.download_leaves())
        except Exception as e:  # reported, never fatal for the GPU number
            cpub = {"error": repr(e)}
    stats = plan1.stats()
    line = {
        "metric": METRIC, "value": value if ok else None, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS.get(cfg.name, cfg.name), "n": int(cfg.n), "mode": mode,
                   "dag": plan1.dag_mode, "executor": args.exec, "rank_cap": rc,
                   "step": "one H-LU factorization of the config matrix (one k_persistent launch)",
                   "parallelism": "single GPU" if world == 1 else f"replicas x{world} (one matrix per GPU)",
                   "l2": ("inputs larger than L2 (A pool %.0f MB)" % (A0.store.values.numel() * 8 / 2**20)
                          if big else "flushed by a 256 MiB write before every timed step"),
                   "tasks": stats["tasks"], "ops": stats["ops"], "waves": stats["waves"]},
        "factor_time_s": t_ms * 1e-3,
        "factor_time_steps_s": [x * 1e-3 for x in per_step],
        "gflop_per_factorization": flops / 1e9,
        "truncations": c["truncations"],
        "parity": par,
        "roofline": roofline,
        "cpu_baseline": cpub,
        "e2e": e2e,
        "batched": batched,
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
        "setup": setup,
    }
    if not ok:
        line["value_withheld"] = "factors failed the parity check against the reference fixture"
        line["value_unchecked"] = value
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
    rc = rank_cap_of("c4", args.rank_cap)
    t0 = time.time()
    batch = InstanceBatch(ids, rank_cap=rc)
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
    # parity: every instance's L/U ranks vs the reference fixtures that exist
    from tests.golden_inputs import have, load

    rl, ru = batch.ranks()
    checked, bad = 0, 0
    for b, j in enumerate(ids):
        if have(f"c4_{j}"):
            _, arr = load(f"c4_{j}")
            sel = arr["std_L_rank"] >= 0
            bad += int((rl[b][sel] != arr["std_L_rank"][sel]).sum() + (ru[b][sel] != arr["std_U_rank"][sel]).sum())
            checked += 1
    t = float(np.mean(ms))
    tot = torch.tensor([t, flops, bad], dtype=torch.float64, device="cuda")
    if dist is not None:
        tmax = tot[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        fl = tot[1:].clone()
        dist.all_reduce(fl, op=dist.ReduceOp.SUM)
        t, flops_all, bad = float(tmax.item()), float(fl[0].item()), int(fl[1].item())
    else:
        flops_all = flops
    if rank == 0:
        peaks = fp64_peaks(torch)
        ach = flops / (float(np.mean(ms)) * 1e-3) / 1e12
        value = flops_all / (t * 1e-3) / 1e9
        line = {"metric": METRIC, "value": value if bad == 0 else None, "unit": "GFLOP/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": WORKLOADS["c4"], "instances": args.instances,
                           "instances_per_gpu": len(ids), "rank_cap": rc,
                           "step": "all instances of this GPU's shard in one k_persistent launch",
                           "parallelism": f"instances sharded x{world}",
                           "l2": "flushed by a 256 MiB write before every timed step"},
                "parity": {"instances_with_reference_fixture": checked, "rank_mismatches": bad},
                "roofline": {"bound": "tensor", "achieved": ach, "peak": peaks["dgemm_tflops"],
                             "unit": "TFLOP/s", "frac": ach / peaks["dgemm_tflops"],
                             "traffic": load_profile_traffic("c4"),
                             "peak_source": "FP64: torch/cuBLAS DGEMM measured in this run",
                             "kernel": "k_persistent (one launch = the shard's instances)"},
                "gpu_launches": args.steps, "clocks": clk.summary(),
                "setup": {"assembly_and_plan_s": setup_s}}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

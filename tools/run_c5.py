"""Config 5 end to end on one GPU: structure, rank-first device assembly
with rank-bounded arenas, native lowering with accumulator-storage reuse,
one accumulator H-LU (the merged DAG's tasks), probe residual
||A x - L U x|| / ||A x||.   python tools/run_c5.py [c5] [acc_budget_GB]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1911_07531_b200 import configs, hmatrix as H  # noqa: E402
from paper_1911_07531_b200.accumulator import AccumulatorMap, hlu_accu  # noqa: E402

def run(name="c5", acc_gb=32.0, log=print):
    """One accumulator H-LU of a large config; returns the report dict."""
    mult = float(os.environ.get("HMX_CAP_MULT", "2.5"))
    floor = int(os.environ.get("HMX_CAP_FLOOR", "24"))
    retries = int(os.environ.get("HMX_C5_RETRY", "0"))
    want_trace = bool(os.environ.get("HMX_C5_TRACE"))
    # 148 per-CTA arenas at the 99.99th percentile of the task needs (166 MB for c5)
    # + 7 peak-size arenas under the 48 GB scratch budget
    os.environ.setdefault("HMX_SCRATCH_PCT", "99.99")
    out = {"config": name}
    cfg = configs.config(name)
    t0 = time.time()
    _, _, perm, broot = configs.structure(cfg)
    pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
    t1 = time.time()
    out["structure_s"] = t1 - t0
    from paper_1911_07531_b200 import _lib  # noqa: E402
    from paper_1911_07531_b200.arith import clear_plans, get_plan  # noqa: E402

    X = np.random.default_rng(7).normal(size=(cfg.n, 2))
    for attempt in range(1 + retries):
        t1 = time.time()
        A, caps = H.assemble_bounded(broot, configs.kernel(cfg, perm), pol, rank_cap=128, mult=mult, floor=floor)
        torch.cuda.synchronize()
        t2 = time.time()
        out.update(attempt=attempt, cap_mult=mult, cap_floor=floor, assembly_s=t2 - t1,
                   A_pool_gb=A.store.values.numel() * 8 / 2**30)
        log(json.dumps(out), flush=True)
        AX = np.asarray(H.hm_apply(A, X))
        L, U = H.zeros(broot, pol, 128, caps), H.zeros(broot, pol, 128, caps)
        kw = dict(acc_budget=int(acc_gb * 2**30 / 8), scratch_budget=int(float(os.environ.get("HMX_C5_SCRATCH_GB", "48")) * 2**30), split_min=0)
        torch.cuda.empty_cache()  # plan_create allocates with cudaMalloc: release torch's cached blocks
        out.update(mem_before_plan_gb=torch.cuda.memory_allocated() / 2**30,
                   mem_reserved_gb=torch.cuda.memory_reserved() / 2**30)
        t3 = time.time()
        plan = get_plan(A.table, "accu", pol, 128, split_min=0, caps=caps, acc_budget=kw["acc_budget"],
                        scratch_budget=kw["scratch_budget"])
        t4 = time.time()
        st = plan.stats()
        out.update(plan_s=t4 - t3, plan=st, plan_scratch_small_mb=plan.plan.scratch_doubles * 8 / 2**20,
                   plan_scratch_big_mb=plan.plan.big_doubles * 8 / 2**20, n_big=plan.plan.n_big,
                   mem_after_plan_gb=torch.cuda.memory_allocated() / 2**30)
        log(json.dumps(out), flush=True)
        H.counters.reset()
        if want_trace:
            plan.plan.enable_trace(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        status = 0
        try:
            hlu_accu(A, L, U, AccumulatorMap(), pol, **kw)
        except _lib.HmxError as e:
            status = int(e.code)
            out["error"] = str(e)
        e1.record()
        torch.cuda.synchronize()
        c = plan.counters()
        lr, ur = L.store.ranks.cpu().numpy(), U.store.ranks.cpu().numpy()
        sel = A.table.leaf & A.table.adm
        at_cap = int(((np.maximum(lr, ur) >= caps) & sel).sum())
        out.update(status=status, factor_s=e0.elapsed_time(e1) / 1e3, gflop=c["flops"] / 1e9,
                   gflops=c["flops"] / (e0.elapsed_time(e1) * 1e-3) / 1e9, truncations=c["truncations"],
                   L_rank_max=int(lr[sel].max()), U_rank_max=int(ur[sel].max()),
                   leaves_at_cap=at_cap, cap_min_slack=int((caps[sel] - np.maximum(lr[sel], ur[sel])).min()),
                   peak_mem_gb=torch.cuda.max_memory_allocated() / 2**30)
        # probe residual ||A x - L U x|| / ||A x|| (also for a clipped run: it measures the clipping)
        res = float(np.linalg.norm(AX - np.asarray(H.hm_apply(L, np.asarray(H.hm_apply(U, X)))))
                    / np.linalg.norm(AX))
        out["probe_residual"] = res
        if status == 0:
            out.pop("error", None)
        if want_trace:
            st_, en_, _sm = plan.plan.trace()
            dur = (en_ - st_) / 1e3
            prof = plan.plan.op_profile
            names = {1: "GEMM", 2: "COPY", 3: "ZERO", 4: "ADD", 5: "LU", 6: "TRSM_LL", 7: "TRSM_UT", 8: "TRUNC",
                     9: "D2LR", 10: "SETRANK", 11: "APPEND", 12: "tr.QR", 13: "svd.RRQR", 14: "svd.Jacobi",
                     15: "tr.recomp"}
            out["op_busy_s"] = {names.get(c_, str(c_)): [float(prof[c_, 0]) / 1e9, int(prof[c_, 1])]
                                for c_ in range(16) if prof[c_, 1]}
            out["busy_sum_s"] = float(dur.sum() / 1e6)
            out["span_s"] = float((en_.max() - st_.min()) / 1e9)
            top = np.argsort(-dur)[:12]
            ops = plan.prog.ops
            tk = []
            for t_ in top:
                o_ = ops[plan.prog.task_ops[t_]:plan.prog.task_ops[t_ + 1]]
                big = [(int(x["code"]), int(x["dim"][0]), int(x["dim"][1])) for x in o_ if x["code"] in (8, 9)]
                tk.append([float(dur[t_] / 1e3), len(o_), big[:4]])
            out["slowest_tasks_ms"] = tk
            out["tasks_over_10ms"] = int((dur > 1e4).sum())
            out["tasks_over_100ms"] = int((dur > 1e5).sum())
        log(json.dumps(out), flush=True)
        if status == 0 or not (status & 8):
            break
        # rank overflow: repeat with larger bounds
        del A, L, U, plan
        clear_plans()
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        mult *= 1.6
    os.makedirs("gpurun_out", exist_ok=True)
    return out


if __name__ == "__main__":
    run(sys.argv[1] if len(sys.argv) > 1 else "c5", float(sys.argv[2]) if len(sys.argv) > 2 else 32.0)

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

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
acc_gb = float(sys.argv[2]) if len(sys.argv) > 2 else 32.0
mult = float(os.environ.get("HMX_CAP_MULT", "2.5"))
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
for attempt in range(3):
    t1 = time.time()
    A, caps = H.assemble_bounded(broot, configs.kernel(cfg, perm), pol, rank_cap=128, mult=mult)
    torch.cuda.synchronize()
    t2 = time.time()
    out.update(attempt=attempt, cap_mult=mult, assembly_s=t2 - t1,
               A_pool_gb=A.store.values.numel() * 8 / 2**30)
    print(json.dumps(out), flush=True)
    AX = np.asarray(H.hm_apply(A, X))
    L, U = H.zeros(broot, pol, 128, caps), H.zeros(broot, pol, 128, caps)
    kw = dict(acc_budget=int(acc_gb * 2**30 / 8), scratch_budget=int(24 * 2**30), split_min=0)
    t3 = time.time()
    plan = get_plan(A.table, "accu", pol, 128, split_min=0, caps=caps, acc_budget=kw["acc_budget"],
                    scratch_budget=kw["scratch_budget"])
    t4 = time.time()
    st = plan.stats()
    out.update(plan_s=t4 - t3, plan=st, plan_scratch_small_mb=plan.plan.scratch_doubles * 8 / 2**20,
               plan_scratch_big_mb=plan.plan.big_doubles * 8 / 2**20, n_big=plan.plan.n_big,
               mem_after_plan_gb=torch.cuda.memory_allocated() / 2**30)
    print(json.dumps(out), flush=True)
    H.counters.reset()
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
    if status == 0:
        res = float(np.linalg.norm(AX - np.asarray(H.hm_apply(L, np.asarray(H.hm_apply(U, X)))))
                    / np.linalg.norm(AX))
        out["probe_residual"] = res
        out.pop("error", None)
    print(json.dumps(out), flush=True)
    if status == 0 or not (status & 8):
        break
    # rank overflow: repeat with larger bounds
    del A, L, U, plan
    clear_plans()
    torch.cuda.empty_cache()
    mult *= 1.6
os.makedirs("gpurun_out", exist_ok=True)

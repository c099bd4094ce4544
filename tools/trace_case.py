"""Per-task device timeline of one H-LU: where the time goes.

python tools/trace_case.py [config] [mode] [exec]
Prints time by task kind, the slowest tasks, and the critical path of the
execution graph weighted by measured task durations.
"""
import sys, os, time, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_07531_b200 import configs, hmatrix as H, engine
from paper_1911_07531_b200.arith import get_plan

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
mode = sys.argv[2] if len(sys.argv) > 2 else None
exe = int(sys.argv[3]) if len(sys.argv) > 3 else engine.EXEC_PERSISTENT
cfg = configs.config(name)
mode = mode or cfg.mode
geom, root, perm, broot = configs.structure(cfg)
pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
RC = 128 if name.startswith("c5") else 64
A0 = H.assemble(broot, configs.kernel(cfg, perm), pol, rank_cap=RC)
split = int(os.environ.get("HMX_SPLIT", "256"))
plan = get_plan(A0.table, mode, pol, RC, split_min=split)
A = A0.copy(); L = H.zeros(broot, pol, RC); U = H.zeros(broot, pol, RC)
plan.run(A.store, L.store, U.store, exe)
A.store.copy_from(A0.store)
plan.plan.enable_trace(True)
torch.cuda.synchronize()
t0 = time.time()
plan.run(A.store, L.store, U.store, exe)
torch.cuda.synchronize()
wall = time.time() - t0
st, en, sm = plan.plan.trace()
dur = (en - st) / 1e3  # us
span = (en.max() - st.min()) / 1e6
kinds = np.array(plan.prog.kinds)
names = {1:"GEMM",2:"COPY",3:"ZERO",4:"ADD",5:"LU",6:"TRSM_LL",7:"TRSM_UT",8:"TRUNC",9:"D2LR",10:"SETRANK",11:"APPEND",
         12:"tr.QR", 13:"svd.RRQR", 14:"svd.Jacobi(n=sweeps)", 15:"tr.recomp"}
prof = plan.plan.op_profile
for code in range(16):
    if prof[code, 1]:
        print(f"  op {names.get(code, code):8s} n={prof[code,1]:8d} busy={prof[code,0]/1e6:9.2f} ms mean={prof[code,0]/prof[code,1]/1e3:8.1f} us")
print(f"{name} {mode} exec={exe}: wall {wall*1e3:.1f} ms, device span {span:.1f} ms, tasks {len(dur)}")
print("busy sum %.1f ms -> mean parallelism %.1f" % (dur.sum() / 1e3, dur.sum() / 1e3 / span))
for k in sorted(set(kinds)):
    d = dur[kinds == k]
    print(f"  {k:14s} n={len(d):6d} sum={d.sum()/1e3:9.2f} ms mean={d.mean():9.1f} us max={d.max():9.1f} us")
nops = np.diff(plan.prog.task_ops)
idx = np.argsort(-dur)[:15]
for i in idx:
    print(f"  slow: {plan.prog.keys[i]} {dur[i]:.0f} us ops={nops[i]}")
# critical path with measured durations
ptr, sidx = plan.succ_ptr, plan.succ_idx
n = len(dur)
fin = np.zeros(n)
for t in range(n):  # program order is topological
    pass
best = dur.copy()
pred = -np.ones(n, dtype=np.int64)
order = np.arange(n)
finish = dur.copy()
for t in range(n):
    for j in sidx[ptr[t]:ptr[t + 1]]:
        if finish[t] + dur[j] > finish[j]:
            finish[j] = finish[t] + dur[j]
            pred[j] = t
end = int(np.argmax(finish))
print("critical path (measured durations): %.1f ms" % (finish[end] / 1e3))
path = []
while end >= 0:
    path.append(end); end = pred[end]
path = path[::-1]
from collections import Counter
c = Counter(); cd = Counter()
for t in path:
    c[kinds[t]] += 1; cd[kinds[t]] += dur[t]
print("  path length", len(path), {k: (c[k], round(cd[k] / 1e3, 2)) for k in c})
# op-code histogram on the critical path
ops = plan.prog.ops
oc = Counter()
for t in path:
    for o in ops[plan.prog.task_ops[t]:plan.prog.task_ops[t + 1]]:
        oc[int(o["code"])] += 1
print("  ops on path", dict(oc))
# exact per-op time on the critical path (per-op device durations)
opt = plan.plan.op_times
pc, pn = Counter(), Counter()
for t in path:
    a, b = plan.prog.task_ops[t], plan.prog.task_ops[t + 1]
    for i in range(a, b):
        code = int(ops[i]["code"])
        key = names.get(code, code)
        if code == 8:
            K = int(ops[i]["dim"][0])
            kin = int(plan.plan.op_inner[i])
            kb = 16 if kin <= 16 else 32 if kin <= 32 else 64 if kin <= 64 else 128 if kin <= 128 else 256 if kin <= 256 else 4096
            key = f"TRUNC m={K} K<={kb}"
        if code == 9:
            key = f"D2LR m={int(ops[i]['dim'][0])}"
        pc[key] += opt[i] / 1e3
        pn[key] += 1
print("  critical-path time by op:")
for k, v in pc.most_common(24):
    print(f"    {k:16s} {v/1e3:8.2f} ms  n={pn[k]}")
pd = sorted(path, key=lambda t: -dur[t])[:25]
for t in pd:
    o = ops[plan.prog.task_ops[t]:plan.prog.task_ops[t + 1]]
    tr = [(int(x["dim"][0]), int(x["dim"][1])) for x in o if x["code"] in (8, 9)]
    print(f"  path task {plan.prog.keys[t]} {dur[t]:.0f}us ops={len(o)} trunc/d2lr={tr}")

"""Busy-time histogram of TRUNC / GEMM / D2LR by resolved shape for one H-LU.

python tools/op_hist.py [config]
Sum over all CTAs (what bounds batched throughput), not the critical path.
"""
import os
import sys
from collections import defaultdict

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1911_07531_b200 import configs, engine, hmatrix as H  # noqa: E402
from paper_1911_07531_b200.arith import get_plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = configs.config(name)
geom, root, perm, broot = configs.structure(cfg)
pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
A0 = H.assemble(broot, configs.kernel(cfg, perm), pol, rank_cap=64)
plan = get_plan(A0.table, cfg.mode, pol, 64)
A = A0.copy(); L = H.zeros(broot, pol, 64); U = H.zeros(broot, pol, 64)
plan.run(A.store, L.store, U.store, engine.EXEC_PERSISTENT)
A.store.copy_from(A0.store)
plan.plan.enable_trace(True)
plan.run(A.store, L.store, U.store, engine.EXEC_PERSISTENT)
torch.cuda.synchronize()
plan.plan.trace()
ops = plan.prog.ops
t = plan.plan.op_times / 1e3  # us
kin = plan.plan.op_inner


def bucket(x):
    return 1 << int(np.ceil(np.log2(max(int(x), 1))))


for code, label in ((8, "TRUNC"), (1, "GEMM"), (9, "D2LR")):
    sel = np.nonzero(ops["code"] == code)[0]
    agg = defaultdict(lambda: [0, 0.0])
    for i in sel:
        m, n = int(ops["dim"][i, 0]), int(ops["dim"][i, 1])
        if m < 0 or n < 0:
            m, n = -1, -1
        key = (m, n, bucket(kin[i]) if code != 9 else 0)
        agg[key][0] += 1
        agg[key][1] += t[i]
    tot = sum(v[1] for v in agg.values())
    print(f"{label}: n={len(sel)} busy={tot / 1e3:.1f} ms")
    for k, (cnt, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
        print(f"   m={k[0]:5d} n={k[1]:5d} K<={k[2]:4d}  n={cnt:7d}  busy={s / 1e3:8.1f} ms "
              f"({100 * s / tot:4.1f}%)  mean={s / cnt:7.1f} us")

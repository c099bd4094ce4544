"""One warm c2 accumulator factorization (for ncu): setup, 1 warm-up, then
`--reps` factorizations through the persistent executor."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1911_07531_b200 import configs, engine, hmatrix as H  # noqa: E402
from paper_1911_07531_b200.arith import get_plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = configs.config(name)
geom, root, perm, broot = configs.structure(cfg)
pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
A0 = H.assemble(broot, configs.kernel(cfg, perm), pol, rank_cap=64)
plan = get_plan(A0.table, cfg.mode, pol, 64)
A = A0.copy()
L, U = H.zeros(broot, pol, 64), H.zeros(broot, pol, 64)
for i in range(1 + reps):
    A.store.copy_from(A0.store)
    torch.cuda.synchronize()
    plan.run(A.store, L.store, U.store, engine.EXEC_PERSISTENT)
torch.cuda.synchronize()
print("ok", plan.counters())

"""Where does a c5_d3 factorization spend its time: host stack every 120 s."""
import faulthandler
import sys
import time

faulthandler.dump_traceback_later(120, repeat=True)
sys.path.insert(0, '.')
import torch  # noqa: E402

from paper_1911_07531_b200 import configs, engine, hmatrix as H  # noqa: E402
from paper_1911_07531_b200.arith import get_plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5_d3"
cfg = configs.config(name)
geom, root, perm, broot = configs.structure(cfg)
pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
t0 = time.time()
A0 = H.assemble(broot, configs.kernel(cfg, perm), pol, rank_cap=128)
torch.cuda.synchronize()
print("assembled", time.time() - t0, flush=True)
plan = get_plan(A0.table, cfg.mode, pol, 128)
print("planned", time.time() - t0, plan.stats(), flush=True)
A = A0.copy(); L = H.zeros(broot, pol, 128); U = H.zeros(broot, pol, 128)
t1 = time.time()
plan.run(A.store, L.store, U.store, engine.EXEC_PERSISTENT, check=False)
torch.cuda.synchronize()
print("factorized", time.time() - t1, "status", plan.plan.status(), plan.counters(), flush=True)

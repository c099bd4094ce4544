"""Rank-first device assembly of a config (default c5) and a dump of its
ranks: python tools/c5_assemble.py [c5] [outdir]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1911_07531_b200 import configs, hmatrix as H  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
cfg = configs.config(name)
t0 = time.time()
_, _, perm, broot = configs.structure(cfg)
t1 = time.time()
pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
A, caps = H.assemble_bounded(broot, configs.kernel(cfg, perm), pol, rank_cap=128)
torch.cuda.synchronize()
t2 = time.time()
r = A.store.ranks.cpu().numpy()
t = A.table
sel = t.leaf & t.adm
print(f"{name}: structure {t1 - t0:.1f}s assembly {t2 - t1:.1f}s; pool {A.store.values.numel() * 8 / 2**30:.2f} GB; "
      f"ranks: max {r[sel].max()} mean {r[sel].mean():.1f}; peak mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GB",
      flush=True)
for m in sorted(set(t.m[sel].tolist())):
    s2 = sel & (t.m == m)
    print(f"  blocks {m}: {s2.sum()} ranks max {r[s2].max()} mean {r[s2].mean():.1f}")
os.makedirs(out, exist_ok=True)
np.savez_compressed(os.path.join(out, f"{name}_A_ranks.npz"), ranks=r)

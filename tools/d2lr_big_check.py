"""dense_to_lowrank of blocks with a large revealed rank (the shapes of c5 /
c5_d3: eps = 1e-4, capacity 128) against the oracle; one case per argument
"m,n,sep" or the default list.  python tools/d2lr_big_check.py [m,n,sep ...]"""
import sys
import time

import numpy as np

sys.path.insert(0, '.')
import torch  # noqa: E402

from oracle.hm_oracle import Policy, dense_to_lowrank as ref  # noqa: E402
from paper_1911_07531_b200 import kernels  # noqa: E402
from tests.test_kernels_gpu import _Pol, _kernel_block  # noqa: E402

cases = [tuple(float(x) for x in a.split(",")) for a in sys.argv[1:]] or [
    (128, 128, 0.05), (128, 128, 0.01), (256, 256, 0.1), (256, 128, 0.05), (512, 512, 0.15), (512, 512, 0.05),
    (1024, 1024, 0.25)]
import os
eps = float(os.environ.get('EPS', '1e-4'))
for (m, n, sep) in cases:
    m, n = int(m), int(n)
    M = _kernel_block(m, n, sep, m + n)
    s = np.linalg.svd(M, compute_uv=False)
    k8 = int((s > 1e-4 * eps * s[0]).sum())
    Ur, Vr = ref(M, Policy("accuracy", eps=eps))
    print(f"{m}x{n} sep {sep}: rank ref {Ur.shape[1]} sv>1e-8: {k8} ...", end="", flush=True)
    torch.cuda.synchronize()
    t0 = time.time()
    Un, Vn = kernels.dense_to_lowrank(M, _Pol("accuracy", eps=eps), cap=min(m, n, 128))
    torch.cuda.synchronize()
    dt = time.time() - t0
    x = np.random.default_rng(0).normal(size=(n, 2))
    err = np.linalg.norm(Un @ (Vn.T @ x) - Ur @ (Vr.T @ x)) / np.linalg.norm(Ur @ (Vr.T @ x))
    print(f" dev {Un.shape[1]}  wall {dt*1e3:.1f} ms  err {err:.2e}", flush=True)

"""Per-block parity diagnostics of a device factorization vs the reference
fixture: relative Frobenius differences of A (input), L and U per block,
against the block's norm relative to the matrix.  python tools/parity_diag.py c3 [accu]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1911_07531_b200 import configs, hmatrix as H  # noqa: E402
from paper_1911_07531_b200.accumulator import AccumulatorMap, hlu_accu  # noqa: E402
from paper_1911_07531_b200.arith import hlu  # noqa: E402
from tests import parity as PT  # noqa: E402
from tests.golden_inputs import load  # noqa: E402

name = sys.argv[1]
mode = sys.argv[2] if len(sys.argv) > 2 else "accu"
meta, arr = load(name)
cfg = configs.config(name)
_, _, perm, broot = configs.structure(cfg)
pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
rc = 128 if name.startswith("c5") else 64
A = H.assemble(broot, configs.kernel(cfg, perm), pol, rank_cap=rc)
lay = A.store.layout
fa = PT.store_fro(lay, A.store.values.cpu().numpy(), A.store.ranks.cpu().numpy())
L, U = H.zeros(broot, pol, rc), H.zeros(broot, pol, rc)
(hlu if mode == "std" else lambda *a: hlu_accu(a[0], a[1], a[2], AccumulatorMap(), a[3]))(A, L, U, pol)
out = {}
for tag, f, ref in (("A", fa, arr["A_fro"]),
                    ("L", PT.store_fro(lay, L.store.values.cpu().numpy(), L.store.ranks.cpu().numpy()), arr[f"{mode}_L_fro"]),
                    ("U", PT.store_fro(lay, U.store.values.cpu().numpy(), U.store.ranks.cpu().numpy()), arr[f"{mode}_U_fro"])):
    sel = np.isfinite(ref) & np.isfinite(f) & (ref > 0)
    rel = np.abs(f[sel] - ref[sel]) / ref[sel]
    tot = np.sqrt(np.nansum(ref[sel] ** 2))
    scale = ref[sel] / tot
    absn = np.abs(f[sel] - ref[sel]) / tot
    i = int(np.argmax(rel))
    uids = np.flatnonzero(sel)
    print(f"{tag}: blocks {sel.sum()}  rel max {rel.max():.3e} q99 {np.quantile(rel, .99):.3e} q50 {np.median(rel):.3e}"
          f"  | worst uid {uids[i]} size {lay.table.m[uids[i]]}x{lay.table.nc[uids[i]]} ref {ref[uids[i]]:.3e} (block/total {scale[i]:.2e})"
          f"  | abs/total max {absn.max():.3e}")
    for thr in (1e-8, 1e-6, 1e-4):
        big = scale > thr
        if big.any():
            print(f"     blocks with norm > {thr:g} of the total: {big.sum()}, rel max {rel[big].max():.3e}")

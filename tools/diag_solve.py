import sys, numpy as np
sys.path.insert(0, '.')
from tests.test_ops_gpu import setup, ranks
from oracle import hm_oracle as O
from paper_1911_07531_b200 import hmatrix as H, arith
A, pol, eps, broot, hpol = setup()
L, U, _, _ = O.factor(A, "std", pol)
for cap in (128, None):
    M = A.copy(); X = O.zeros(A.bt)
    O.htrsl(L, 0, M, 0, X, pol)
    dT = H.from_leaves(broot, L.lv, hpol, cap); dM = H.from_leaves(broot, A.lv, hpol, cap); dX = H.zeros(broot, hpol, cap)
    arith.htrsl(dT, dM, dX, hpol)
    got = ranks(dX.store.download_leaves(), A.bt); ref = ranks(X.lv, A.bt)
    d = np.nonzero(got != ref)[0]
    print("cap", cap, "mismatch", len(d), [(int(u), int(got[u]), int(ref[u]), A.bt.shape(u)) for u in d[:10]])

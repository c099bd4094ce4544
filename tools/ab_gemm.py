"""GEMM op latency/throughput of the loaded libhmx (HMX_LIB selects an A/B
build): batched m x n x k products through hmx_gemm_batched, one CTA per
product.  python tools/ab_gemm.py [m n k batch]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1911_07531_b200 import _lib  # noqa: E402

shapes = [(64, 64, 64), (128, 128, 64), (64, 64, 256), (256, 256, 256), (128, 32, 128)]
if len(sys.argv) > 3:
    shapes = [tuple(int(x) for x in sys.argv[1:4])]
batch = 148 * 4
L = _lib.lib()
for m, n, k in shapes:
    A = torch.randn(batch, k, m, dtype=torch.float64, device="cuda")
    B = torch.randn(batch, n, k, dtype=torch.float64, device="cuda")
    C = torch.zeros(batch, n, m, dtype=torch.float64, device="cuda")
    ts = []
    for r in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.hmx_gemm_batched(batch, m, n, k, 1.0, _lib.ptr(A), m, m * k, 0, _lib.ptr(B), k, k * n, 0,
                                      0.0, _lib.ptr(C), m, m * n, _lib.stream_ptr()), "gemm")
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts[1:])
    ref = torch.bmm(A.transpose(1, 2), B.transpose(1, 2))
    err = float((C.transpose(1, 2) - ref).abs().max() / ref.abs().max())
    print(f"GEMM {m}x{n}x{k} batch {batch}: {t * 1e3 / batch * 148:.1f} us per CTA-op, "
          f"{2 * m * n * k * batch / (t * 1e-3) / 1e12:.3f} TFLOP/s, max rel err {err:.1e}", flush=True)

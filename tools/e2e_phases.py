"""Phase times of the e2e leg (batch.PipelinedHLU) on c2, R replicas:
H2D of packed A, unpack, factorization, pack of L and U, D2H; and the
pipelined per-step time at several K (fill/drain amortisation)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1911_07531_b200 import engine, hmatrix as H  # noqa: E402
from paper_1911_07531_b200.batch import PipelinedHLU  # noqa: E402

R = int(os.environ.get("R", "16"))
cfg, broot, pol, A0, setup = bench.build_case("c2", 64)
AB0 = H.HBatch.replicate(A0, R)
hA_v, hA_r = AB0.download_packed()
torch.cuda.synchronize()
hA_v, hA_r = hA_v.clone().pin_memory(), hA_r.clone().pin_memory()
del AB0
torch.cuda.empty_cache()
pipe = PipelinedHLU(broot, pol, R, 64, cfg.mode, engine.EXEC_PERSISTENT)
res, ev = pipe.run([(hA_v, hA_r)] * 3)
torch.cuda.synchronize()
pipe.check()
outs = [res[0], res[1]]
A, L, U = pipe.sets[0]
buf = A._xfer_buf()


def t(fn, s, n=3):
    ms = []
    for _ in range(n):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        with torch.cuda.stream(s):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return min(ms)


s = pipe.s_comp
print("packed A GB", hA_v.numel() * 8 / 1e9, "L,U GB", [o[0].numel() * 8 / 1e9 for o in outs[0]])
print("h2d ms", t(lambda: buf[:hA_v.numel()].copy_(hA_v, non_blocking=True), pipe.s_h2d))
print("unpack ms", t(lambda: A.store.unpack_from(buf, stream=s), s))
A.store.unpack_from(buf, stream=s)
torch.cuda.synchronize()
print("run ms", t(lambda: pipe.plan.run(A.store, L.store, U.store, engine.EXEC_PERSISTENT, s, check=False), s, 1))
for k, M in enumerate((L, U)):
    print(f"pack{k} ms", t(lambda: M.store.pack_to(M._xfer_buf(), pipe.offs[0][k], stream=s), s))
hv = outs[0][0][0]
n = hv.numel()
print("d2h ms (L)", t(lambda: hv.copy_(L._xfer_buf()[:n], non_blocking=True), pipe.s_d2h))
for K in (2, 5, 10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(pipe.s_h2d)
    res, ev = pipe.run([(hA_v, hA_r)] * K, [outs[i & 1] for i in range(K)])
    e1.record(pipe.s_d2h)
    torch.cuda.synchronize()
    print(f"pipelined K={K}: ms/step", e0.elapsed_time(e1) / K, flush=True)

"""Latency of single device ops (one CTA per op, batch <= #SMs).

python tools/bench_kernels.py
Times OP_TRUNC / OP_D2LR / OP_GEMM / OP_LU / TRSM on representative shapes
of the c2 op trace, through an hmx plan executed repeatedly (plan creation
outside the timed region).  Reports microseconds per op (= per CTA).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1911_07531_b200 import _lib  # noqa: E402

SB = _lib.SCRATCH_BASE


def run(ops_per_task, bases, scratch, reps=5, nt=None, trace=False):
    nt = len(ops_per_task)
    ops = np.concatenate(ops_per_task)
    task_ops = np.zeros(nt + 1, np.int64)
    task_ops[1:] = np.cumsum([len(x) for x in ops_per_task])
    plan = _lib.Plan(ops, task_ops, np.zeros(nt + 1, np.int32), np.zeros(0, np.int32),
                     np.array([0, nt], np.int32), np.arange(nt, dtype=np.int32), scratch, 4)
    for b, (v, r) in bases.items():
        plan.bind(b, v, r)
    if trace:
        plan.enable_trace(True)
    plan.execute(0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        plan.reset_counters()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.execute(0)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    st = plan.status()
    prof = None
    if trace:
        plan.trace()
        prof = plan.op_profile
    plan.close()
    return min(ts), st, prof


def trunc_case(m, n, K, decay=0.3, eps=1e-6, batch=int(os.environ.get('HMX_BENCH_BATCH', '148')), trace=False):
    rng = np.random.default_rng(0)
    kb = max(K, int(os.environ.get('HMX_BENCH_KB', '0')))
    U = rng.normal(size=(batch, K, m)) * np.exp(-decay * np.arange(K))[None, :, None]
    V = rng.normal(size=(batch, K, n))
    dU = torch.from_numpy(U.reshape(batch, -1)).cuda()
    dV = torch.from_numpy(V.reshape(batch, -1)).cuda()
    out = torch.zeros(batch, (m + n) * K, dtype=torch.float64, device="cuda")
    rk = torch.zeros(batch, dtype=torch.int32, device="cuda")
    offV = m * kb
    offW = offV + n * kb
    scratch = offW + 9 * kb * kb + (m + n + 200) * kb + 2048
    tasks = []
    for b in range(batch):
        o = np.zeros(3, dtype=_lib.OP_DTYPE)
        o[0]["code"] = _lib.OP_COPY; o[0]["dim"][:2] = (m, K); o[0]["farg"][0] = 1.0
        o[0]["ref"][0] = _lib.mref(0, b * m * K); o[0]["ld"][0] = m
        o[0]["ref"][2] = _lib.mref(SB, 0); o[0]["ld"][2] = m
        o[1]["code"] = _lib.OP_COPY; o[1]["dim"][:2] = (n, K); o[1]["farg"][0] = 1.0
        o[1]["ref"][0] = _lib.mref(1, b * n * K); o[1]["ld"][0] = n
        o[1]["ref"][2] = _lib.mref(SB, offV); o[1]["ld"][2] = n
        t = o[2]
        t["code"] = _lib.OP_TRUNC; t["dim"][:3] = (m, n, K)
        t["ref"][0] = _lib.mref(SB, 0); t["ld"][0] = m
        t["ref"][1] = _lib.mref(SB, offV); t["ld"][1] = n
        t["ref"][2] = _lib.mref(2, b * (m + n) * K); t["ld"][2] = m
        t["ref"][3] = _lib.mref(2, b * (m + n) * K + m * K); t["ld"][3] = n
        t["wref"] = _lib.mref(SB, offW)
        t["slot"][0] = _lib.slot(3, b)
        t["iarg"][:4] = (2, 0, K, kb)
        t["farg"][1] = eps
        tasks.append(o)
    us, st, prof = run(tasks, {0: (dU, None), 1: (dV, None), 2: (out, None), 3: (None, rk)},
                       scratch, trace=trace)
    return us, st, float(rk.float().mean().item()), prof


def d2lr_case(m, n, decay=0.15, eps=1e-6, batch=int(os.environ.get('HMX_BENCH_BATCH', '148'))):
    rng = np.random.default_rng(1)
    # 2D exp-kernel block between neighbouring boxes (realistic numerical rank)
    g = int(np.sqrt(m))
    if g * (m // g) == m:
        a = np.stack(np.meshgrid(np.arange(g), np.arange(m // g), indexing="ij"), -1).reshape(-1, 2) / 128
    else:  # random points in a box of the same density
        a = rng.random((m, 2)) * (g / 128.0)
    b = a + np.array([g / 128.0 * 1.5, 0.0])
    d = np.linalg.norm(a[:, None, :] - b[None, :n, :], axis=-1)
    M = np.exp(-d / 0.2)  # smooth spectrum: the revealed rank is the numerical rank
    Ms = np.stack([M.T.ravel() * (1 + 1e-3 * b) for b in range(batch)])
    dM = torch.from_numpy(Ms).cuda()
    out = torch.zeros(batch, (m + n) * min(m, n), dtype=torch.float64, device="cuda")
    rk = torch.zeros(batch, dtype=torch.int32, device="cuda")
    l = max(m, n)
    scratch = m * n + 8 * l + (3 * l * l + 2500000 if l >= 256 else 16 * l * l)
    tasks = []
    for b in range(batch):
        o = np.zeros(2, dtype=_lib.OP_DTYPE)
        o[0]["code"] = _lib.OP_COPY; o[0]["dim"][:2] = (m, n); o[0]["farg"][0] = 1.0
        o[0]["ref"][0] = _lib.mref(0, b * m * n); o[0]["ld"][0] = m
        o[0]["ref"][2] = _lib.mref(SB, 0); o[0]["ld"][2] = m
        t = o[1]
        t["code"] = _lib.OP_D2LR; t["dim"][:2] = (m, n)
        t["ref"][0] = _lib.mref(SB, 0); t["ld"][0] = m
        t["ref"][2] = _lib.mref(2, b * (m + n) * min(m, n)); t["ld"][2] = m
        t["ref"][3] = _lib.mref(2, b * (m + n) * min(m, n) + m * min(m, n)); t["ld"][3] = n
        t["wref"] = _lib.mref(SB, m * n)
        t["slot"][0] = _lib.slot(3, b)
        t["iarg"][:3] = (2, 0, min(m, n, 64))
        t["farg"][1] = eps
        tasks.append(o)
    us, st, prof = run(tasks, {0: (dM, None), 2: (out, None), 3: (None, rk)}, scratch, trace=True)
    return us, st, float(rk.float().mean().item()), prof


def dshapes_only():
    return any(a.startswith("d") for a in sys.argv[1:]) and not any("," in a and not a.startswith("d") for a in sys.argv[1:])


def main():
    names = {12: "QR", 13: "RRQR", 14: "Jacobi", 15: "recomp"}
    shapes = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:] if "," in a and not a.startswith("d")]
    for (m, n, K) in shapes or ([] if dshapes_only() else [(64, 64, 20), (64, 64, 40), (128, 128, 24), (256, 256, 24), (256, 256, 48),
                      (512, 512, 30), (1024, 1024, 30), (1024, 1024, 120), (2048, 2048, 30)]):
        us, st, r, prof = trunc_case(m, n, K, trace=True)
        ph = " ".join(f"{names[c]}={prof[c,0]/max(prof[c,1],1)/1e3:.0f}us" for c in (12, 13, 15))
        sw = prof[14, 1] / max(prof[13, 1], 1)
        print(f"TRUNC m={m:5d} n={n:5d} K={K:4d}: {us:9.1f} us/op  rank~{r:.1f} status={st} "
              f"[{ph} Jacobi={prof[14,0]/max(prof[13,1],1)/1e3:.0f}us sweeps={sw:.1f}]", flush=True)
    dshapes = [tuple(int(x) for x in a[1:].split(",")) for a in sys.argv[1:] if a.startswith("d")]
    for (m, n) in (dshapes if (shapes or dshapes) else [(64, 64), (128, 128), (256, 256), (512, 512)]):
        us, st, r, prof = d2lr_case(m, n)
        nd = max(prof[9, 1], 1)
        ph = " ".join(f"{names[c]}={prof[c,0]/nd/1e3:.0f}us" for c in (12, 13, 14, 15))
        print(f"D2LR  m={m:5d} n={n:5d}: {us:9.1f} us/op  rank~{r:.1f} status={st} [{ph} sweeps={prof[14,1]/nd:.1f}]", flush=True)


if __name__ == "__main__":
    main()

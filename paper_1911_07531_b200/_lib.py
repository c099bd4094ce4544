"""ctypes binding of libhmx.so (include/hmx.h).

The product path has no CPU fallback: importing the engine on a machine
without the built library raises, and every device entry point raises
``HmxError`` when the library reports a failure.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._build import LIB as _BUILT_LIB

# HMX_LIB: load another in-tree build of the same sources (A/B experiments)
LIB = os.environ.get("HMX_LIB") or _BUILT_LIB

# op codes (hmx_engine.cu)
OP_NOP, OP_GEMM, OP_COPY, OP_ZERO, OP_ADD, OP_LU, OP_TRSM_LL, OP_TRSM_UT = range(8)
OP_TRUNC, OP_D2LR, OP_SETRANK, OP_APPEND, OP_SVALS, OP_TRSM_UN = 8, 9, 10, 11, 12, 13
F_TA, F_TB, F_ACC = 1, 2, 4
SCRATCH_BASE = 15

HMX_OK = 0
HMX_ERR_ARG, HMX_ERR_CUDA, HMX_ERR_PIVOT = 1, 2, 4
HMX_ERR_RANK_OVERFLOW, HMX_ERR_NOT_CONVERGED, HMX_ERR_TIMEOUT = 8, 16, 32

POLICY_EXACT, POLICY_RANK, POLICY_ACCURACY = 0, 1, 2

OP_DTYPE = np.dtype([
    ("code", "<i4"), ("flags", "<i4"), ("dim", "<i4", 4), ("ld", "<i4", 4),
    ("ref", "<i8", 4), ("slot", "<i4", 4), ("iarg", "<i4", 4), ("farg", "<f8", 2),
    ("wref", "<i8"),
])
assert OP_DTYPE.itemsize == 128


class HmxError(RuntimeError):
    def __init__(self, code, what=""):
        self.code = int(code)
        names = [n for b, n in ((1, "bad argument"), (2, "CUDA error"), (4, "singular pivot"),
                                (8, "rank overflow"), (16, "Jacobi not converged"),
                                (32, "scheduler timeout")) if self.code & b]
        super().__init__(f"hmx {what}: status {self.code} ({', '.join(names) or 'ok'})")


def d2lr_scratch(m: int, n: int) -> int:
    """Workspace (doubles) an OP_D2LR of an m x n block needs (op.wref): the
    warp-synchronous / global pivoted-QR paths of hmx_engine.cu keep their
    reflector blocks, R1^T, the fat core's scratch and (blocks of 256 and
    more) a copy of the block there.  hmx_lower.cpp uses the same formula."""
    l = max(int(m), int(n))
    return 8 * l + (3 * l * l + 2500000 if l >= 256 else 16 * l * l)


def trunc_scratch(m: int, n: int, kb: int) -> int:
    """Workspace (doubles) of an OP_TRUNC with stacked capacity kb."""
    kb = max(int(kb), 1)
    return 9 * kb * kb + (int(m) + int(n) + 200) * kb + 2048


def mref(base: int, off: int) -> int:
    return (int(base) << 56) | int(off)


def slot(base: int, idx: int) -> int:
    return -(1 + ((int(base) << 24) | int(idx)))


class _PlanDesc(C.Structure):
    _fields_ = [
        ("ops", C.c_void_p), ("n_ops", C.c_int64),
        ("task_ops", C.c_void_p), ("n_tasks", C.c_int32),
        ("succ_ptr", C.c_void_p), ("succ_idx", C.c_void_p),
        ("wave_ptr", C.c_void_p), ("wave_tasks", C.c_void_p), ("n_waves", C.c_int32),
        ("scratch_doubles", C.c_int64), ("scratch_ranks", C.c_int32), ("max_ctas", C.c_int32),
        ("ctas_per_sm", C.c_int32),
        ("task_scratch", C.c_void_p), ("big_scratch_doubles", C.c_int64), ("n_big", C.c_int32),
    ]


_lib = None


def lib():
    """Load libhmx.so; raise if it is missing (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        raise RuntimeError(f"libhmx.so not built at {LIB}; run __graft_entry__.build()")
    L = C.CDLL(LIB)
    vp, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "hmx_version": ([], C.c_char_p),
        "hmx_op_workspace": ([i32, i32, i32, i32], i64),
        "hmx_op_size": ([], C.c_int),
        "hmx_getrf_nopiv_batched": ([i32, i32, vp, i32, i64, vp, vp, i64, vp, vp], i32),
        "hmx_trsm_lower_unit_batched": ([i32, i32, i32, vp, i32, i64, vp, i32, i64, vp], i32),
        "hmx_trsm_upper_trans_batched": ([i32, i32, i32, vp, i32, i64, vp, i32, i64, vp], i32),
        "hmx_trsm_upper_batched": ([i32, i32, i32, vp, i32, i64, vp, i32, i64, vp], i32),
        "hmx_gemm_batched": ([i32, i32, i32, i32, f64, vp, i32, i64, i32, vp, i32, i64, i32, f64,
                              vp, i32, i64, vp], i32),
        "hmx_truncate_batched": ([i32, i32, i32, i32, vp, vp, i64, i64, i32, i32, f64, i32, vp, vp,
                                  i64, i64, vp, vp], i32),
        "hmx_dense_to_lowrank_batched": ([i32, i32, i32, vp, i64, i32, i32, f64, i32, vp, vp, i64,
                                          i64, vp, vp], i32),
        "hmx_svd_values_batched": ([i32, i32, i32, vp, i64, vp, i64, vp], i32),
        "hmx_plan_create": ([C.POINTER(_PlanDesc), C.POINTER(vp)], i32),
        "hmx_plan_bind": ([vp, i32, vp, vp], i32),
        "hmx_plan_execute": ([vp, i32, vp], i32),
        "hmx_plan_status": ([vp, vp, C.POINTER(i32)], i32),
        "hmx_plan_counters": ([vp, vp, C.POINTER(C.c_uint64)], i32),
        "hmx_plan_reset_counters": ([vp, vp], i32),
        "hmx_plan_destroy": ([vp], i32),
        "hmx_plan_trace": ([vp, i32, vp], i32),
        "hmx_exp_kernel_blocks": ([i32, vp, vp, i32, vp, f64, f64, f64, vp, vp], i32),
        "hmx_fp64_fma_probe": ([i32, i32, vp, vp], i32),
        "hmx_plan_partition": ([vp, i32, i32, vp, vp, vp, i64], i32),
        "hmx_plan_sched_state": ([vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)], i32),
        "hmx_plan_peer": ([vp, i32, vp, vp, vp, vp, vp], i32),
        "hmx_plan_reset": ([vp, vp], i32),
        "hmx_ipc_handle": ([vp, vp, C.POINTER(i64)], i32),
        "hmx_ipc_open": ([vp, C.POINTER(vp)], i32),
        "hmx_ipc_close": ([vp], i32),
        "hmx_pack_leaves": ([i32, i32, vp, i64, i32, vp, vp, vp, i64, vp, vp], i32),
        "hmx_unpack_leaves": ([i32, i32, vp, i64, i32, vp, vp, vp, vp, vp], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    if L.hmx_op_size() != OP_DTYPE.itemsize:
        raise RuntimeError("libhmx.so op record size mismatch")
    _lib = L
    return L


EXPORTED = (
    "hmx_version", "hmx_op_size", "hmx_op_workspace", "hmx_getrf_nopiv_batched", "hmx_trsm_lower_unit_batched",
    "hmx_trsm_upper_trans_batched", "hmx_trsm_upper_batched", "hmx_gemm_batched", "hmx_truncate_batched",
    "hmx_dense_to_lowrank_batched", "hmx_svd_values_batched", "hmx_plan_create",
    "hmx_plan_bind", "hmx_plan_execute", "hmx_plan_status", "hmx_plan_counters",
    "hmx_plan_reset_counters", "hmx_plan_destroy", "hmx_plan_trace", "hmx_exp_kernel_blocks", "hmx_fp64_fma_probe",
    "hmx_plan_partition", "hmx_plan_sched_state", "hmx_plan_peer", "hmx_plan_reset",
    "hmx_ipc_handle", "hmx_ipc_open", "hmx_ipc_close", "hmx_pack_leaves", "hmx_unpack_leaves",
)


def ipc_handle(ptr):
    """(64-byte CUDA IPC handle of the allocation holding device address
    ptr, ptr's byte offset in it)."""
    h = (C.c_uint8 * 64)()
    off = C.c_int64()
    check(lib().hmx_ipc_handle(C.c_void_p(int(ptr)), h, C.byref(off)), "ipc_handle")
    return bytes(h), int(off.value)


def ipc_open(handle: bytes):
    """Map a peer allocation; returns its base address in this process."""
    h = (C.c_uint8 * 64).from_buffer_copy(handle)
    base = C.c_void_p()
    check(lib().hmx_ipc_open(h, C.byref(base)), "ipc_open")
    return int(base.value)


def ipc_close(base):
    check(lib().hmx_ipc_close(C.c_void_p(int(base))), "ipc_close")


def check(status, what=""):
    if status != HMX_OK:
        raise HmxError(status, what)


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


class Plan:
    """Owning handle of a device execution plan (hmx_plan_t)."""

    def __init__(self, ops, task_ops, succ_ptr, succ_idx, wave_ptr, wave_tasks,
                 scratch_doubles, scratch_ranks, max_ctas=0, ctas_per_sm=1, task_scratch=None,
                 n_big=0, scratch_budget=None):
        """task_scratch (per-task need, doubles) enables tiered scratch: each
        CTA gets an arena at the 99.9th percentile of the needs; tasks above
        it share peak-size arenas, one per 4 CTAs (n_big=0) or n_big.
        scratch_budget (bytes, large problems): the per-CTA arenas of all
        CTAs take at most half of it and the peak-size arenas the other
        half (at least one)."""
        L = lib()
        big, ts = 0, None
        if task_scratch is not None and len(task_scratch):
            ts = np.ascontiguousarray(task_scratch, dtype=np.int64)
            peak = int(ts.max())
            small = max(int(np.percentile(ts, float(os.environ.get("HMX_SCRATCH_PCT", "99.9")))), 1 << 16)
            if scratch_budget:
                nct = (max_ctas or 148 * max(1, int(ctas_per_sm)))
                small = min(small, max(1 << 16, int(scratch_budget) // 2 // 8 // nct))
                if peak > small:
                    n_big = max(1, int(scratch_budget) // 2 // 8 // peak)
            if peak > small:
                scratch_doubles = small
                big = peak
                n_big = int(n_big) if n_big else -4
                if n_big > 0:
                    n_big = int(min(int((ts > small).sum()), n_big))
            else:
                scratch_doubles = max(peak, 1)
                n_big = 0
        self._keep = [np.ascontiguousarray(ops, dtype=OP_DTYPE),
                      np.ascontiguousarray(task_ops, dtype=np.int64),
                      np.ascontiguousarray(succ_ptr, dtype=np.int32),
                      np.ascontiguousarray(succ_idx, dtype=np.int32),
                      np.ascontiguousarray(wave_ptr, dtype=np.int32),
                      np.ascontiguousarray(wave_tasks, dtype=np.int32)]
        o, to, sp, si, wp, wt = self._keep
        d = _PlanDesc(o.ctypes.data, len(o), to.ctypes.data, len(to) - 1, sp.ctypes.data,
                      si.ctypes.data, wp.ctypes.data, wt.ctypes.data, len(wp) - 1,
                      int(scratch_doubles), int(scratch_ranks), int(max_ctas), int(ctas_per_sm),
                      ts.ctypes.data if ts is not None else None, int(big), int(n_big))
        self.scratch_doubles, self.big_doubles, self.n_big = int(scratch_doubles), int(big), int(n_big)
        h = C.c_void_p()
        check(L.hmx_plan_create(C.byref(d), C.byref(h)), "plan_create")
        self.h = h
        self._keep = None
        self.n_tasks = len(to) - 1
        self.n_ops = len(o)

    def bind(self, base_id, values, ranks=None):
        check(lib().hmx_plan_bind(self.h, int(base_id), ptr(values), ptr(ranks)), "plan_bind")

    def partition(self, nranks, rank, owner, pub_ptr, pub):
        """Attach a block-row partition (hmx_plan_partition)."""
        o = np.ascontiguousarray(owner, dtype=np.int32)
        pp = np.ascontiguousarray(pub_ptr, dtype=np.int64)
        pb = np.ascontiguousarray(pub)
        check(lib().hmx_plan_partition(self.h, int(nranks), int(rank), o.ctypes.data, pp.ctypes.data,
                                       pb.ctypes.data if len(pb) else None, len(pb)), "plan_partition")

    def sched_state(self):
        a, b, c = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib().hmx_plan_sched_state(self.h, C.byref(a), C.byref(b), C.byref(c)), "sched_state")
        return int(a.value or 0), int(b.value or 0), int(c.value or 0)

    def peer(self, r, bases, rbases, indeg, queue, qctl):
        """Storage (16 pool + 16 rank-array addresses) and scheduler state of rank r."""
        bb = (C.c_void_p * 16)(*[int(x or 0) for x in bases])
        rb = (C.c_void_p * 16)(*[int(x or 0) for x in rbases])
        check(lib().hmx_plan_peer(self.h, int(r), bb, rb, C.c_void_p(int(indeg)), C.c_void_p(int(queue)),
                                  C.c_void_p(int(qctl))), "plan_peer")

    def reset(self, stream=None):
        check(lib().hmx_plan_reset(self.h, stream_ptr(stream)), "plan_reset")

    def execute(self, mode=2, stream=None):
        check(lib().hmx_plan_execute(self.h, int(mode), stream_ptr(stream)), "plan_execute")

    def status(self, stream=None) -> int:
        v = C.c_int32()
        check(lib().hmx_plan_status(self.h, stream_ptr(stream), C.byref(v)), "plan_status")
        return int(v.value)

    def counters(self, stream=None):
        arr = (C.c_uint64 * 4)()
        check(lib().hmx_plan_counters(self.h, stream_ptr(stream), arr), "plan_counters")
        return [int(x) for x in arr]

    def reset_counters(self, stream=None):
        check(lib().hmx_plan_reset_counters(self.h, stream_ptr(stream)), "plan_reset")

    def enable_trace(self, on=True):
        check(lib().hmx_plan_trace(self.h, int(bool(on)), None), "plan_trace")

    def trace(self):
        out = np.zeros(3 * self.n_tasks + 32 + self.n_ops, dtype=np.uint64)
        check(lib().hmx_plan_trace(self.h, 1, out.ctypes.data_as(C.c_void_p)), "plan_trace")
        t = out[:3 * self.n_tasks].reshape(-1, 3)
        self.op_profile = out[3 * self.n_tasks:3 * self.n_tasks + 32].reshape(16, 2).astype(np.int64)
        w = out[3 * self.n_tasks + 32:]
        self.op_times = (w & np.uint64((1 << 40) - 1)).astype(np.int64)
        self.op_inner = (w >> np.uint64(40)).astype(np.int64)  # resolved K of GEMM/TRUNC
        return t[:, 0].astype(np.int64), t[:, 1].astype(np.int64), (t[:, 2] & 0xffffffff).astype(np.int64)

    def close(self):
        if getattr(self, "h", None):
            lib().hmx_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

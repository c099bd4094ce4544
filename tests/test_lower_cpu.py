"""Native H-LU lowering (csrc/hmx_lower.cpp) vs the Python planner.

planner.py states the lowering of arith.hlu / accumulator.hlu_accu to
device op programs; the native planner must produce the same op records
(byte for byte), task table, scratch sizes, accumulator and workspace
layouts, and the same execution graph against the reference DAG."""

import numpy as np
import pytest

from paper_1911_07531_b200 import configs, engine, hmatrix as H, lower, planner, taskgraph as tg
from paper_1911_07531_b200.trees import BlockTable

CASES = [("s1", "std", 0), ("s1", "accu", 0), ("s2", "std", 0), ("s2", "accu", 0),
         ("s2", "std", 256), ("s2", "accu", 256), ("c1", "std", 0), ("c4_0", "std", 0),
         ("c4_0", "accu", 0), ("s5", "accu", 256), ("c2", "accu", 256)]


def _table(name):
    cfg = configs.config(name)
    _, _, _, broot = configs.structure(cfg)
    return cfg, BlockTable(broot)


@pytest.mark.parametrize("name,mode,split", CASES)
def test_native_lowering_equals_python(name, mode, split):
    cfg, t = _table(name)
    pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
    p = planner.plan_hlu(t, mode, pol, 64, split_min=split)
    q = lower.NativeProgram(t, mode, pol, 64, split_min=split)
    assert len(p.ops) == len(q.ops)
    assert p.ops.tobytes() == q.ops.tobytes()
    assert np.array_equal(p.task_ops, q.task_ops)
    assert np.array_equal(p.task_scratch, q.task_scratch)
    assert (p.scratch_doubles, p.scratch_ranks, p.acc_size, p.ws_size, p.ws_slots, p.updates) == \
        (q.scratch_doubles, q.scratch_ranks, q.acc_size, q.ws_size, q.ws_slots, q.updates)
    assert [k for k in p.keys if k[0] != "micro"] == [k for k in q.keys if k[0] != "micro"]
    for f in ("d_off", "u_off", "v_off", "cap"):
        assert np.array_equal(getattr(p.layout, f), getattr(q.layout, f))
    assert p.layout.size == q.layout.size
    # execution graph: Python ExecPlan._exec_graph vs the native one
    dm = "std" if mode == "std" else "accu-merged"

    class _P:
        pass

    f = _P()
    f.prog, f.mode, f.table = p, mode, t
    f.dag = tg.build_dag_native(t, dm)
    ptr, idx, _, _ = engine.ExecPlan._exec_graph(f)
    h = tg.dag_handle(t, dm)
    p2, i2 = q.graph(h.ptr, mode)
    h.free()
    assert np.array_equal(ptr, p2) and np.array_equal(idx, i2)


def test_native_lowering_rank_bounded_layout():
    """Per-block capacity bounds shrink the low-rank arenas (N4) and every
    reference to them; without bounds the layout is the rank_cap one."""
    cfg, t = _table("s2")
    pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
    q0 = lower.NativeProgram(t, "accu", pol, 64)
    caps = np.full(t.n, -1, np.int32)
    caps[t.adm & t.leaf] = 8
    q1 = lower.NativeProgram(t, "accu", pol, 64, caps=caps)
    assert q1.layout.size < q0.layout.size
    sel = t.adm & t.leaf
    assert (q1.layout.cap[sel] == np.minimum(q0.layout.cap[sel], 8)).all()
    assert len(q1.ops) == len(q0.ops)


def test_native_lowering_errors():
    """A low-rank diagonal block cannot be factored (hmatrix.py:322-323)."""
    cfg, t = _table("s1")
    pol = H.TruncationPolicy.fixed_accuracy(cfg.eps)
    bad = BlockTable(t.root)
    bad.adm = bad.adm.copy()
    bad.adm[bad.leaf & (bad.r0 == bad.c0)] = True
    with pytest.raises(ValueError):
        lower.NativeProgram(bad, "std", pol, 64)

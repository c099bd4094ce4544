"""Lowered programs vs the reference DAG (CPU): task sets, execution
graphs and the soundness of the reference DAG as a schedule."""

import numpy as np
import pytest

from oracle.hm_oracle import Policy
from paper_1911_07531_b200 import configs, planner, taskgraph as tg
from paper_1911_07531_b200.trees import BlockTable


def case(name):
    cfg = configs.config(name)
    _, _, _, broot = configs.structure(cfg)
    return cfg, BlockTable(broot)


class _P:
    pass


def exec_graph(prog, dag, mode, table):
    from paper_1911_07531_b200.engine import ExecPlan

    ep = _P()
    ep.prog, ep.dag, ep.mode, ep.table = prog, dag, mode, table
    return ExecPlan._exec_graph(ep)


@pytest.mark.parametrize("name", ["s1", "s2"])
@pytest.mark.parametrize("mode,dag_mode", [("std", "std"), ("accu", "accu-merged")])
def test_tasks_are_dag_nodes_and_graph_is_ordered(name, mode, dag_mode):
    cfg, bt = case(name)
    prog = planner.plan_hlu(bt, mode, Policy("accuracy", eps=cfg.eps), rank_cap=64)
    dag = tg.build_hlu_dag(bt, dag_mode)
    keys = {(t.kind, t.uids, t.alpha) for t in dag.nodes}
    assert keys == set(prog.keys)
    ptr, idx, n_dag, _ = exec_graph(prog, dag, mode, bt)
    src = np.repeat(np.arange(len(prog.keys)), np.diff(ptr))
    assert (src < idx).all()  # program (sequential) order is a topological order
    lv = tg.asap_levels(len(prog.keys), ptr, idx)
    assert lv.max() >= 1


def _reach(n, ptr, idx):
    reach = [0] * n
    for u in range(n - 1, -1, -1):
        r = 0
        for v in idx[ptr[u]:ptr[u + 1]]:
            r |= (1 << int(v)) | reach[int(v)]
        reach[u] = r
    return reach


@pytest.mark.parametrize("name", ["s1"])
def test_std_dag_implies_every_data_dependency(name):
    """SPEC.md 'refinement soundness': every hazard of the sequential
    program is ordered by a path of the reference's std DAG."""
    cfg, bt = case(name)
    prog = planner.plan_hlu(bt, "std", Policy("accuracy", eps=cfg.eps), rank_cap=64)
    dag = tg.build_hlu_dag(bt, "std")
    ptr, idx, _, _ = exec_graph(prog, dag, "std", bt)
    reach = _reach(len(prog.keys), ptr, idx)
    for a, b in planner.dataflow_edges(prog, {i: bt for i in range(4)}):
        assert reach[a] >> b & 1, (prog.keys[a], prog.keys[b])


@pytest.mark.parametrize("name", ["s1", "s2"])
def test_merged_dag_contradicts_accumulator_fold_order(name):
    """Why accumulator plans use data-flow edges: the reference's merged DAG
    orders some add_upd pairs against hlu_accu's program order (a WAW on
    matrix A between nested blocks), so its edge set cannot replay
    hlu_accu's per-accumulator fold sequence (SURVEY.md finding 3)."""
    cfg, bt = case(name)
    prog = planner.plan_hlu(bt, "accu", Policy("accuracy", eps=cfg.eps), rank_cap=64)
    dag = tg.build_hlu_dag(bt, "accu-merged")
    pos = {k: i for i, k in enumerate(prog.keys)}
    back = [(u.kind, v.kind) for u, v in dag.edges()
            if pos[(u.kind, u.uids, u.alpha)] > pos[(v.kind, v.uids, v.alpha)]]
    assert all(k == ("add_upd", "add_upd") for k in back)
    if name == "s2":
        assert back  # the 2D structure exhibits it


def test_replicate_shifts_refs_and_slots():
    cfg, bt = case("s1")
    prog = planner.plan_hlu(bt, "std", Policy("accuracy", eps=cfg.eps), rank_cap=64)
    lay = prog.layout
    sizes = {0: lay.size, 1: lay.size, 2: lay.size, 3: prog.acc_size}
    slots = {i: bt.n for i in range(4)}
    ops, to, nt = planner.replicate(prog, 3, sizes, slots)
    n = len(prog.ops)
    assert len(ops) == 3 * n and to[-1] == 3 * n and len(to) == 3 * nt + 1
    m56 = (1 << 56) - 1
    for i in range(0, n, 7):
        for c in range(3):
            a, b = prog.ops[i], ops[c * n + i]
            for r0, r1 in zip(a["ref"], b["ref"]):
                base = int(r0) >> 56
                if base in sizes:
                    assert (int(r1) & m56) == (int(r0) & m56) + c * sizes[base]
                else:
                    assert r1 == r0


def test_wavefront_batches_group_by_op_type_and_leaf_shape():
    """engine.wave_batches: the ASAP wavefronts stay intact and inside every
    wavefront tasks of equal signature (op type, leaf shape) are contiguous."""
    from paper_1911_07531_b200 import taskgraph as tg
    from paper_1911_07531_b200.engine import wave_batches

    cfg, bt = case("s2")
    prog = planner.plan_hlu(bt, "accu", Policy("accuracy", eps=cfg.eps), rank_cap=64)
    nt = len(prog.task_ops) - 1
    from paper_1911_07531_b200.planner import dataflow_edges

    e = np.array(sorted(dataflow_edges(prog, {0: bt, 1: bt, 2: bt})), dtype=np.int64).reshape(-1, 2)
    ptr = np.zeros(nt + 1, dtype=np.int32)
    np.add.at(ptr, e[:, 0] + 1, 1)
    ptr = np.cumsum(ptr).astype(np.int32)
    idx = e[np.argsort(e[:, 0], kind="stable"), 1].astype(np.int32)
    lv = tg.asap_levels(nt, ptr, idx)
    order, sig = wave_batches(lv, prog.ops, prog.task_ops)
    assert sorted(order.tolist()) == list(range(nt))
    lo = lv[order]
    assert (np.diff(lo) >= 0).all()
    so = sig[order]
    same = np.diff(lo) == 0
    assert (np.diff(so)[same] >= 0).all()          # sorted inside a wavefront: batches are contiguous
    nb = len(np.unique(np.stack([lo, so], 1), axis=0))
    assert nb < nt                                   # tasks do share batches
    # a truncating task is keyed by its truncation: op code 8 or 9 in the signature
    codes = set((so >> 44).tolist())
    assert codes & {8, 9}

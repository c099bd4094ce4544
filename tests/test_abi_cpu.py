"""The C-ABI library loads on a CPU-only machine and exports every entry
point declared in include/hmx.h (no compute calls without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_1911_07531_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    hdr = open(os.path.join(ROOT, "include", "hmx.h")).read()
    return sorted(set(re.findall(r"\b(hmx_[a-z0-9_]+)\s*\(", hdr)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return ctypes.CDLL(_build.LIB)


def test_every_declared_symbol_is_exported(lib):
    names = declared()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_matches_header():
    assert sorted(_lib.EXPORTED) == declared()


def test_version_and_record_size(lib):
    L = _lib.lib()
    assert L.hmx_version().startswith(b"hmx")
    assert L.hmx_op_size() == 128 == _lib.OP_DTYPE.itemsize


def test_sm100a_code_in_library():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_dag_library_exports_its_header():
    hdr = open(os.path.join(ROOT, "include", "hmx_dag.h")).read()
    names = sorted(set(re.findall(r"\b(hmx_dag_[a-z0-9_]+)\s*\(", hdr)))
    assert len(names) == 7
    dl = ctypes.CDLL(_build.build_dag())
    missing = [n for n in names if not hasattr(dl, n)]
    assert not missing, missing


def test_op_workspace_formulas_agree():
    """The planners (Python: _lib.trunc_scratch / d2lr_scratch; native:
    hmx_lower.cpp, checked op for op against the Python planner in
    test_lower_cpu) size the TRUNC / D2LR workspaces with the formulas the
    device paths assume (hmx_op_workspace): a smaller workspace is overrun."""
    from paper_1911_07531_b200 import _lib

    L = _lib.lib()
    for m, n in ((64, 64), (128, 96), (128, 128), (200, 255), (256, 256), (512, 300), (1024, 1024), (4096, 2048)):
        assert L.hmx_op_workspace(_lib.OP_D2LR, m, n, 0) == _lib.d2lr_scratch(m, n)
        for kb in (1, 16, 64, 200):
            assert L.hmx_op_workspace(_lib.OP_TRUNC, m, n, kb) == _lib.trunc_scratch(m, n, kb)
    assert L.hmx_op_workspace(_lib.OP_GEMM, 64, 64, 0) == 0

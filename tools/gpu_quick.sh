# Quick GPU check: selected tests + bench (args: pytest -k expression)
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "${1:-transfer}" > $O/pytest_quick.log 2>&1; echo "pytest rc=$?" >> $O/pytest_quick.log
timeout 900 python bench.py ${2:-} > $O/bench_quick.log 2>&1; echo "bench rc=$?" >> $O/bench_quick.log

# Perf iteration: correctness subset, op latencies, bench (no cpu baseline)
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "${1:-oracle or executors or c2}" > $O/pytest_perf.log 2>&1; echo "pytest rc=$?" >> $O/pytest_perf.log
timeout 600 python tools/bench_kernels.py > $O/bench_kernels.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench_perf.log 2>&1; echo "bench rc=$?" >> $O/bench_perf.log

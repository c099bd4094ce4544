# correctness subset on the default build + A/B of the variants given as args
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "${PYK:-oracle or executors or c2 or transfer}" > $O/pytest_perf.log 2>&1; echo "pytest rc=$?" >> $O/pytest_perf.log
for v in "$@"; do
  lib=paper_1911_07531_b200/libhmx${v}.so
  HMX_LIB=$PWD/$lib timeout 600 python tools/bench_kernels.py > $O/ab_kernels${v}.log 2>&1
  HMX_LIB=$PWD/$lib timeout 900 python bench.py --steps 3 --no-cpu-baseline > $O/ab_bench${v}.log 2>&1
done

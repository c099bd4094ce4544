# A/B/C: op latencies and the bench value for several in-tree builds
cd $GRAFT_REPO_ROOT
O=gpurun_out
for v in "$@"; do
  lib=paper_1911_07531_b200/libhmx${v}.so
  HMX_LIB=$PWD/$lib timeout 600 python tools/bench_kernels.py > $O/ab_kernels${v}.log 2>&1
  HMX_LIB=$PWD/$lib timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > $O/ab_bench${v}.log 2>&1
done

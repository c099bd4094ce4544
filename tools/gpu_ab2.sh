# A/B bench of builds: args = suffixes; env BENCH_ARGS appended
cd $GRAFT_REPO_ROOT
O=gpurun_out
for v in "$@"; do
  lib=paper_1911_07531_b200/libhmx${v}.so
  HMX_LIB=$PWD/$lib timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > $O/ab2_bench${v}.log 2>&1
  HMX_LIB=$PWD/$lib timeout 900 python -m pytest tests/test_hlu_gpu.py -q -x -k "oracle or config_ranks" > $O/ab2_pt${v}.log 2>&1
done

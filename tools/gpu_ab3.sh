# A/B of library variants: bench (c2 batch) + the numerics gates (truncate
# fixtures, kernel tests, c1/c2/c3 rank parity) per variant.  args = suffixes
cd $GRAFT_REPO_ROOT
O=gpurun_out
for v in "$@"; do
  lib=paper_1911_07531_b200/libhmx${v}.so
  HMX_LIB=$PWD/$lib timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > $O/ab3_bench${v}.log 2>&1
  HMX_LIB=$PWD/$lib timeout 600 python tools/bench_kernels.py > $O/ab3_kern${v}.log 2>&1
  HMX_LIB=$PWD/$lib timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_hlu_gpu.py tests/test_dense_ops.py -q -x --durations=5 > $O/ab3_pt${v}.log 2>&1
done
echo done > $O/ab3_done.txt

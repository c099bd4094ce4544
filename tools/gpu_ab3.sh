# A/B of library variants on one box: c2 batch bench + single-op latencies
# per variant (args = suffixes of paper_1911_07531_b200/libhmx<suffix>.so;
# "base" = libhmx.so), then the numerics gates (kernel tests, H-LU rank
# parity c1/c2/c3/c5_d3, dense ops) for the suffixes in $PT_VARIANTS.
cd $GRAFT_REPO_ROOT
O=gpurun_out
libof() { if [ "$1" = "base" ]; then echo "$PWD/paper_1911_07531_b200/libhmx.so"; else echo "$PWD/paper_1911_07531_b200/libhmx$1.so"; fi; }
for v in "$@"; do
  HMX_LIB=$(libof $v) timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-e2e $BENCH_ARGS > $O/ab3_bench_$v.log 2>&1
  HMX_LIB=$(libof $v) timeout 600 python tools/bench_kernels.py > $O/ab3_kern_$v.log 2>&1
done
for v in $PT_VARIANTS; do
  HMX_LIB=$(libof $v) timeout 1500 python -m pytest tests/test_kernels_gpu.py tests/test_hlu_gpu.py tests/test_dense_ops.py -q -x --durations=5 > $O/ab3_pt_$v.log 2>&1
done
echo done > $O/ab3_done.txt

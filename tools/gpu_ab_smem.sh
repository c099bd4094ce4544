#!/bin/bash
# A/B of the 1-CTA/SM shared-memory budget (224 KB default vs 160 KB) on one box, then config 5.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/$1; mkdir -p $O
for cfg in c2 c3; do
  for v in "" _smem160; do
    lib=$PWD/paper_1911_07531_b200/libhmx$v.so
    HMX_LIB=$lib timeout 900 python bench.py --config $cfg --no-cpu-baseline --no-e2e > $O/bench_${cfg}${v}.log 2>&1
  done
done
timeout 3000 python tools/run_c5.py c5 > $O/run_c5.log 2>&1; echo "rc=$?" >> $O/run_c5.log
echo done > $O/done.txt

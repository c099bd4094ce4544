#!/bin/bash
# Closing session of a round: driver-visible bench lines of every config, the reference arm,
# the ncu launch list + one full capture of the dominant kernel, and the DMMA A/B.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/$1; mkdir -p $O
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1800 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "rc=$?" >> $O/bench_c3.err
for cfg in c2 c1 c4 c5_d3; do
  timeout 1200 python bench.py --config $cfg > $O/bench_$cfg.json 2> $O/bench_$cfg.err; echo "rc=$?" >> $O/bench_$cfg.err
done
timeout 1500 python bench.py --impl reference > $O/reference_c3.json 2> $O/reference_c3.err
# DMMA A/B: GEMM op latency / throughput and one c2 factorization with either GEMM variant
# (build the arms first: python tools/build_variant.py _dfma -DHMX_DMMA=0; _dmma -DHMX_DMMA=1)
for v in _dfma _dmma; do
  lib=$PWD/paper_1911_07531_b200/libhmx$v.so
  HMX_LIB=$lib timeout 600 python tools/ab_gemm.py > $O/ab_gemm$v.log 2>&1
  HMX_LIB=$lib timeout 900 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/ab_c2$v.json 2> $O/ab_c2$v.err
done
# A/B: shape-adaptive GEMM tiles in the op interpreter
HMX_LIB=$PWD/paper_1911_07531_b200/libhmx_gwide.so timeout 900 python bench.py --config c3 --no-cpu-baseline --no-e2e > $O/ab_c3_gwide.json 2> $O/ab_c3_gwide.err
HMX_LIB=$PWD/paper_1911_07531_b200/libhmx_gwide.so timeout 900 python bench.py --config c2 --no-cpu-baseline --no-e2e > $O/ab_c2_gwide.json 2> $O/ab_c2_gwide.err
timeout 900 python tools/trace_case.py c2 > $O/trace_c2.txt 2>&1
timeout 900 python tools/trace_case.py c3 > $O/trace_c3.txt 2>&1
# profiler passes (after the plain runs above exited)
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|hmx" --csv \
  --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:k_persistent -s 3 -c 1 -f \
  -o $O/full_c3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
for v in _dfma _dmma; do
  lib=$PWD/paper_1911_07531_b200/libhmx$v.so
  HMX_LIB=$lib timeout 1200 ncu --clock-control none -k regex:k_tasks -c 1 -f \
    --metrics sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__inst_executed.sum \
    --csv --log-file $O/ncu_gemm$v.csv python tools/ab_gemm.py 256 256 256 > $O/ncu_gemm$v.log 2>&1
done
echo done > $O/done.txt

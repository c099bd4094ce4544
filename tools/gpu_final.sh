# Round-end GPU session: full tests, smoke, bench (default), per-config
# single-factorization numbers, executor-variant check, trace, ncu.
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
for c in c1 c4; do timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline > $O/bench_$c.log 2>&1; done
timeout 1200 python bench.py --config c3 --replicas 1 --steps 2 --no-cpu-baseline --no-e2e > $O/bench_c3.log 2>&1
timeout 1200 python bench.py --config c5_d3 --replicas 1 --rank-cap 128 --steps 2 --no-cpu-baseline --no-e2e > $O/bench_c5_d3.log 2>&1
timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-e2e --ctas-per-sm 1 > $O/bench_occ1.log 2>&1
timeout 600 python tools/trace_case.py c2 > $O/trace_c2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_persistent|k_tasks|k_move|k_scan|k_exp_kernel|k_dfma" --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_persistent -s 4 -c 1 \
  -o $O/c2_batch_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
echo done > $O/done.txt

# One GPU session: tests, smoke, bench, per-op profile, ncu launch list and full capture.
cd $GRAFT_REPO_ROOT
O=gpurun_out
nvidia-smi -L > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout 600 python tools/trace_case.py c2 > $O/trace_c2.log 2>&1
timeout 600 python tools/op_hist.py c2 > $O/ophist_c2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_persistent|k_tasks|k_move|k_scan|k_exp_kernel|k_dfma" --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_persistent -s 4 -c 1 \
  -o $O/c2_batch_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
echo done > $O/done.txt

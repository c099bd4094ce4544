# Closing GPU session: full GPU tests, smoke, default bench, reference arm, launch list, ncu full of the step kernel.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${CLOSE_DIR:-close}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_persistent|k_tasks|k_move|k_scan|k_exp_kernel|k_dfma|k_pack|k_unpack" --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_persistent -s 4 -c 1 \
  -o $O/c2_batch_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
echo done > $O/done.txt

cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "dense_ops or transfer or batch" > $O/pytest_rep.log 2>&1; echo "rc=$?" >> $O/pytest_rep.log
for r in 24 32; do
  timeout 900 python bench.py --steps 3 --no-cpu-baseline --no-e2e --replicas $r > $O/rep_bench_$r.log 2>&1
done

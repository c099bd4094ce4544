#!/bin/bash
# One parameterised GPU session (run under gpurun from the repo root).
#   tools/gpu_session.sh OUTDIR STEP [STEP ...]
# Steps:
#   tests            pytest -m gpu
#   smoke            __graft_entry__.smoke()
#   bench[:ARGS]     python bench.py ARGS      (ARGS: comma-separated, e.g. bench:--config,c2)
#   ref[:ARGS]       python bench.py --impl reference ARGS
#   launches[:ARGS]  ncu launch list (gpu__time_duration.sum) of bench.py ARGS
#   ncu[:ARGS]       ncu --set full of one k_persistent launch of bench.py ARGS
#   py:SCRIPT[,ARGS] python SCRIPT ARGS
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/$1
shift
mkdir -p "$O"
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > "$O/smi.txt" 2>&1
for step in "$@"; do
  name=${step%%:*}
  args=""
  [[ "$step" == *:* ]] && args=$(echo "${step#*:}" | tr ',' ' ')
  tag=$name$(echo "$args" | tr -c 'a-zA-Z0-9' '_' | cut -c1-40)
  case $name in
    tests) timeout 2400 python -m pytest tests -m gpu -q $args > "$O/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$O/pytest_gpu.log" ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1; echo "rc=$?" >> "$O/smoke.log" ;;
    bench) timeout 1800 python bench.py $args > "$O/$tag.log" 2>&1; echo "rc=$?" >> "$O/$tag.log" ;;
    ref) timeout 1800 python bench.py --impl reference $args > "$O/$tag.log" 2>&1; echo "rc=$?" >> "$O/$tag.log" ;;
    launches) timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|hmx" --csv \
        --log-file "$O/launches.csv" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e $args \
        > "$O/ncu_launch.log" 2>&1; echo "rc=$?" >> "$O/ncu_launch.log" ;;
    ncu) timeout 2400 ncu --set full --clock-control none --import-source on -k regex:k_persistent -s 4 -c 1 \
        -o "$O/full" python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e $args \
        > "$O/ncu_full.log" 2>&1; echo "rc=$?" >> "$O/ncu_full.log" ;;
    py) timeout 2400 python $args > "$O/$tag.log" 2>&1; echo "rc=$?" >> "$O/$tag.log" ;;
    *) echo "unknown step $name" >> "$O/errors.txt" ;;
  esac
done
echo done > "$O/done.txt"

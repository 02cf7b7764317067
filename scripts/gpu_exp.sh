#!/bin/bash
# experiment loop: build, quick parity, bench lines per config, optional ncu (csv exported on the box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -q -x > gpurun_out/pytest_exp.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_exp.log
for c in ${CONFIGS:-od deca qd dd}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-next > gpurun_out/bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$c.log
done
for c in ${NCU_CONFIGS:-}; do
  ncu -f --set full --clock-control none --import-source on -k regex:conv_ -s ${SKIP:-24} -c 1 -o /tmp/prof_$c python scripts/prof_one.py --config $c --evals 2 > gpurun_out/ncu_full_$c.log 2>&1
  ncu -i /tmp/prof_$c.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$c.csv 2>/dev/null
  ncu -i /tmp/prof_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_$c.csv 2>/dev/null
done
for c in ${LAUNCH_CONFIGS:-}; do
  ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_$c.csv python scripts/prof_one.py --config $c --evals 2 > gpurun_out/ncu_launch_$c.log 2>&1
done
echo done

#!/bin/bash
# round-2 check: GPU tests, smoke, default bench, sweep, launch list of the bench
# command, ncu --set full of the product kernel on od and qd (level 0)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
(nproc; lscpu | grep -i "model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --durations=15 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default.log
timeout 900 python scripts/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1
if [ -z "$SKIP_NCU" ]; then
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-next > gpurun_out/bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-next > gpurun_out/ncu_launch.log 2>&1
for cfg in od qd; do
  skip=8; [ $cfg = qd ] && skip=0
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:conv_ -s $skip -c 1 -o /tmp/prof_$cfg python scripts/prof_one.py --config $cfg --evals 1 > gpurun_out/ncu_full_$cfg.log 2>&1
  ncu -i /tmp/prof_$cfg.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$cfg.csv 2>/dev/null
  ncu -i /tmp/prof_$cfg.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_$cfg.csv 2>/dev/null
  ls -la /tmp/prof_$cfg.ncu-rep >> gpurun_out/ncu_full_$cfg.log
done
fi
echo done

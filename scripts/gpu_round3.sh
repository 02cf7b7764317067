#!/bin/bash
# round-2 final evidence (HEAD after the fused-parts kernel): host facts, smoke, all GPU tests, bench lines (od default,
# dd, qd, deca; reference arm), the launch list of the default bench command,
# ncu --set full of one od and one qd product launch (raw + SASS source CSV),
# executed FP64 counters, the sweep.  Never copies .ncu-rep (64 MiB cap).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
(nproc; lscpu | grep -i "model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv) > gpurun_out/host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --durations=15 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_reference.log
for c in dd qd deca; do timeout 900 python bench.py --config $c --no-next > gpurun_out/bench_$c.log 2>&1; done
if [ -z "$SKIP_NCU" ]; then
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-next > gpurun_out/bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-next > gpurun_out/ncu_launch.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dd.csv python bench.py --config dd --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-next > /dev/null 2>&1
for cfg in od qd; do
  skip=8; [ $cfg = qd ] && skip=0
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:conv_ -s $skip -c 1 -o /tmp/prof_$cfg python scripts/prof_one.py --config $cfg --evals 1 > gpurun_out/ncu_full_$cfg.log 2>&1
  ncu -i /tmp/prof_$cfg.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$cfg.csv 2>/dev/null
  ncu -i /tmp/prof_$cfg.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_$cfg.csv 2>/dev/null
done
for cfg in od qd; do
  skip=8; [ $cfg = qd ] && skip=0
  timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:conv_ -s $skip -c 1 --csv --log-file gpurun_out/fp64_counts_$cfg.csv python scripts/prof_one.py --config $cfg --evals 1 > /dev/null 2>&1
done
fi
timeout 900 python scripts/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1
du -sh gpurun_out
echo done

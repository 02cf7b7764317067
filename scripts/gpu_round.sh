#!/bin/bash
# full round check: smoke, all GPU tests, default bench (cpu_baseline, e2e), reference arm,
# launch list of the bench command, ncu --set full of the product kernel (od)
cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_all.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_reference.log
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
python scripts/prof_one.py --config od --evals 2 > gpurun_out/prof_plain_od.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:conv_ -s 24 -c 1 -o /tmp/prof_conv_od python scripts/prof_one.py --config od --evals 2 > gpurun_out/ncu_full_od.log 2>&1; ncu -i /tmp/prof_conv_od.ncu-rep --page raw --csv > gpurun_out/ncu_raw_od.csv 2>/dev/null; ncu -i /tmp/prof_conv_od.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_od.csv 2>/dev/null; cp /tmp/prof_conv_od.ncu-rep gpurun_out/
echo done

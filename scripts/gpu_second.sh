#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_all.log
python scripts/prof_one.py --config od --evals 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_od.csv python scripts/prof_one.py --config od --evals 2 > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_dig -s 24 -c 1 -o gpurun_out/prof_conv_od python scripts/prof_one.py --config od --evals 2 > gpurun_out/ncu_full.log 2>&1
echo done

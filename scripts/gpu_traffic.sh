#!/bin/bash
# DRAM bytes of every launch of one od evaluation (ncu, cold), the edge tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_edge.py -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_edge.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_edge.log
python scripts/prof_one.py --config od --evals 1 > gpurun_out/traffic_od.log 2>&1 && \
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/traffic_od_step.csv python scripts/prof_one.py --config od --evals 1 >> gpurun_out/traffic_od.log 2>&1
echo done

#!/bin/bash
# NP (part lanes) geometry: tests, tune table on the small-S cells, ncu of the qd product launches
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_geometry.py tests/test_gpu_parity.py -q -x --timeout 300 > gpurun_out/pytest_geom.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_geom.log
TUNE_OUT=gpurun_out/tune_np.json timeout 900 python scripts/tune_table.py qd,sweep_d15_L3,sweep_d15_L4,sweep_d15_L5,sweep_d31_L4,sweep_d31_L5,sweep_d63_L3,sweep_d63_L4,sweep_d63_L5,sweep_d15_L8,sweep_d15_L10,sweep_d31_L8,sweep_d127_L3,sweep_d127_L4,sweep_d127_L5,od > gpurun_out/tune_np.log 2>&1
python scripts/prof_one.py --config qd --evals 1 > gpurun_out/prof_qd.log 2>&1 && \
for s in 0 8; do
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:conv_ -s $s -c 1 -o /tmp/prof_qd_$s python scripts/prof_one.py --config qd --evals 1 > gpurun_out/ncu_qd_$s.log 2>&1
ncu -i /tmp/prof_qd_$s.ncu-rep --page raw --csv > gpurun_out/ncu_raw_qd_$s.csv 2>/dev/null
ncu -i /tmp/prof_qd_$s.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_qd_$s.csv 2>/dev/null
ncu -i /tmp/prof_qd_$s.ncu-rep --page details --csv > gpurun_out/ncu_details_qd_$s.csv 2>/dev/null
done
echo done

#!/bin/bash
# fused-parts kernel, x-streamed build (L >= 8): tests, (F, P, NP) table on the L = 8, 10 cells, ncu of qd fused
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_geometry.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_fused2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fused2.log
TUNE_OUT=gpurun_out/tune_fused2.json timeout 1800 python scripts/tune_table.py ${CELLS:-od,deca,sweep_d15_L8,sweep_d31_L8,sweep_d127_L8,sweep_d15_L10,sweep_d31_L10,sweep_d127_L10} > gpurun_out/tune_fused2.log 2>&1
for G in 2,2,1 2,1,2; do
python scripts/prof_one.py --config qd --evals 1 --geom $G > gpurun_out/prof_qd_$G.log 2>&1 && \
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:conv_ -s 0 -c 1 -o /tmp/p python scripts/prof_one.py --config qd --evals 1 --geom $G > gpurun_out/ncu_qd_$G.log 2>&1
ncu -i /tmp/p.ncu-rep --page raw --csv > gpurun_out/ncu_raw_qd_$G.csv 2>/dev/null
ncu -i /tmp/p.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_qd_$G.csv 2>/dev/null
done
echo done

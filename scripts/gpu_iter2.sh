#!/bin/bash
# iteration check: parity tests of the product kernel, the sweep, ncu raw of qd level 0 and od level 8
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_geometry.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py tests/test_gpu_real.py -q -x --timeout 300 > gpurun_out/pytest_it.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_it.log
timeout 900 python scripts/sweep.py --out gpurun_out/sweep_it.json > gpurun_out/sweep_it.log 2>&1
for cfg in qd od; do
  skip=8; [ $cfg = qd ] && skip=0
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:conv_ -s $skip -c 1 -o /tmp/p_$cfg python scripts/prof_one.py --config $cfg --evals 1 > gpurun_out/ncu_it_$cfg.log 2>&1
  ncu -i /tmp/p_$cfg.ncu-rep --page raw --csv > gpurun_out/ncu_raw_it_$cfg.csv 2>/dev/null
  ncu -i /tmp/p_$cfg.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_it_$cfg.csv 2>/dev/null
done
echo done

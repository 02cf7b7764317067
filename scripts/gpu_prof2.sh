#!/bin/bash
# bench line (od) + dd bench + ncu --set full of od level 8 and qd level 0 (raw + source CSV)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_p2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_p2.log
timeout 300 python bench.py --config dd --no-next --steps 50 > gpurun_out/bench_dd_p2.log 2>&1
timeout 300 python bench.py --config qd --no-next --steps 20 > gpurun_out/bench_qd_p2.log 2>&1
for cfg in od qd; do
  skip=8; [ $cfg = qd ] && skip=0
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:conv_ -s $skip -c 1 -o /tmp/p_$cfg python scripts/prof_one.py --config $cfg --evals 1 > gpurun_out/ncu_p2_$cfg.log 2>&1
  ncu -i /tmp/p_$cfg.ncu-rep --page raw --csv > gpurun_out/ncu_raw_p2_$cfg.csv 2>/dev/null
  ncu -i /tmp/p_$cfg.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_p2_$cfg.csv 2>/dev/null
done
echo done

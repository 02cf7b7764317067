#!/bin/bash
# round-end evidence: the round check plus the sweep at the default algorithm choice
cd $GRAFT_REPO_ROOT
bash scripts/gpu_round.sh
python scripts/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1
python scripts/bench_solve.py > gpurun_out/bench_solve.log 2>&1
echo final-done

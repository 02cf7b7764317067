#!/bin/bash
# first GPU pass: smoke, a parity subset, a short bench
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpuinfo.txt 2>&1
nproc >> gpurun_out/gpuinfo.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "md_ops or ex1 or roundtrip or grid or edge or exact_integer or circle or small_random or dd_full" > gpurun_out/pytest1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest1.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench1.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --algo 1 > gpurun_out/bench1_eft.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench1_eft.log

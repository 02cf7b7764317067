#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "grid or edge or exact_integer or circle or small_random or dd_full or config_sampled" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iter.log
for k in 0 2; do for c in od deca; do
  MDPS_CONV_KERNEL=$k timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_k$k.log 2>&1
done; done

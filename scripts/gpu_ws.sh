#!/bin/bash
# GPU tests on the planned schedule + od/deca time vs workspace bound
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for ws in 0 3000 1000; do
  timeout 300 python bench.py --config od --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-next --workspace-mb $ws > gpurun_out/ws_od_$ws.log 2>&1
done
for ws in 0 3000; do
  timeout 300 python bench.py --config deca --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-next --workspace-mb $ws > gpurun_out/ws_deca_$ws.log 2>&1
done
timeout 300 python bench.py --config qd --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-next > gpurun_out/ws_qd_0.log 2>&1

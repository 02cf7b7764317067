#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python scripts/pdl_ab.py qd,sweep_d15_L4,od > gpurun_out/balance_ab.jsonl 2> gpurun_out/balance_ab.err
for c in qd; do timeout 600 python bench.py --config $c --no-next > gpurun_out/bench_$c.log 2>&1; done
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
echo done

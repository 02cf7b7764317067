#!/bin/bash
# conv kernel variants on the small cells (env MDPS_CONV_KERNEL: 0 two-pass default, 1 Gauss, 2 single pass)
cd $GRAFT_REPO_ROOT
for k in 0 1 2; do
  MDPS_CONV_KERNEL=$k python - <<'PY' > gpurun_out/kind_small_$k.log 2>&1
import json, sys
sys.path.insert(0, "scripts")
import mdinputs
from sweep import measure
for name in ("dd", "qd"):
    print(json.dumps(measure(mdinputs.make_config(name))), flush=True)
for d in (15, 31):
    for L in (2, 3, 4, 5):
        print(json.dumps(measure(mdinputs.sweep_cell(d, L))), flush=True)
PY
done

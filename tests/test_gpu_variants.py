"""The opt-in product-kernel variants (MDPS_CONV_KERNEL = 1 three products per
term, 2 one pass for both parts, 3 two outputs per lane) are
selected once per process, so each runs in a subprocess: a small system at
D = 16, 32, 64 (multiples of 4 for the quad kernel) and a generic odd D,
against the oracle within the tolerance."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import json, sys
sys.path.insert(0, sys.argv[1])
import mdinputs, oracle
from tests.gpu_util import gpu_eval
out = []
for L, degree in ((2, 15), (4, 31), (5, 63), (8, 10)):
    si = mdinputs.random_system(70 + L, n=4, monos=5, m_range=(1, 4), exps=(1, 2), degree=degree, limbs=L)
    v, j, st = gpu_eval(si, 2)
    ov, oj, _ = oracle.eval_diff(si)
    out.append([L, degree, float(max(oracle.series_err(v, ov).max(), oracle.series_err(j, oj).max()))])
print(json.dumps(out))
'''
TOL = {2: 1e-29, 3: 1e-45, 4: 1e-61, 5: 1e-77, 8: 1e-124, 10: 1e-156}


@pytest.mark.parametrize("kind", ("1", "2", "3"))
def test_variant_matches_oracle(kind):
    env = dict(os.environ, MDPS_CONV_KERNEL=kind)
    r = subprocess.run([sys.executable, "-c", CODE, ROOT], env=env, cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    for L, degree, err in json.loads(r.stdout.strip().splitlines()[-1]):
        assert err <= TOL[L], (kind, L, degree, err)

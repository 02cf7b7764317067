"""The work counts behind the roofline:

* W(D, L) — one DFMA per kept digit pair — counted by walking the digit
  product's loop structure (every output k, every term i <= k, both output
  parts, the two real products of a part, the kept triangle u + l <= S - 1)
  equals the closed form D(D+1) S(S+1) that libmdps reports per product
  (`mdps_system_stats`, GPU test) and that bench.py divides by;
* the hardware counters of a profiled launch (ncu, committed under profiles/)
  execute that count within 2% (carries and the output conversion are the
  excess), and the algorithmic share of all executed FP64 instructions is
  above 90% (od) / 85% (qd)."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def digits_for(L):
    S = 2
    while (S - 2) * 23 < 53 * L + 8:
        S += 1
    return S


def walk_digit_dfma(D, S):
    n = 0
    for k in range(D):
        for i in range(k + 1):
            for part in range(2):
                for prod in range(2):
                    for l in range(S):
                        for u in range(S - l):
                            n += 1
    return n


@pytest.mark.parametrize("D,L", [(1, 2), (9, 3), (16, 4), (17, 5), (32, 8)])
def test_walk_equals_closed_form(D, L):
    S = digits_for(L)
    assert walk_digit_dfma(D, S) == D * (D + 1) * S * (S + 1)


def test_digits_per_limb_count():
    # the digit counts DESIGN.md §6 states: (S - 2) * 23 >= 53 L + 8
    assert [digits_for(L) for L in (2, 3, 4, 5, 8, 10)] == [7, 10, 12, 14, 21, 26]


def test_profiled_counters_match_the_algorithmic_count():
    prof = json.load(open(os.path.join(ROOT, "profiles", "r02_fp64_counts.json")))
    seen = set()
    for c in prof["launches"]:
        S = digits_for({"od": 8, "qd": 4}[c["config"]])
        assert c["S"] == S
        assert c["W_algorithmic_dfma"] == c["jobs"] * c["D"] * (c["D"] + 1) * S * (S + 1)
        assert 1.0 <= c["dfma_executed"] / c["W_algorithmic_dfma"] <= 1.02
        assert c["algorithmic_share_of_fp64"] >= {"od": 0.90, "qd": 0.85}[c["config"]]
        seen.add(c["config"])
    assert seen == {"od", "qd"}


@pytest.mark.gpu
@pytest.mark.parametrize("D,L", [(16, 4), (33, 8), (64, 10)])
def test_library_reports_the_walked_count(D, L):
    import mdinputs
    import paper_2012_06607_b200 as mdps
    si = mdinputs.random_system(640 + D + L, n=3, monos=3, m_range=(2, 3), exps=(1,), degree=D - 1, limbs=L)
    with mdps.System.from_inputs(si, algo=mdps.MDPS_ALGO_DIGITS) as s:
        st = s.stats()
    assert st["fp64_ops_conv"] == st["products"] * walk_digit_dfma(D, digits_for(L))

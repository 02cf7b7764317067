"""Stall reasons per code region of an ncu source-page (SASS) CSV: the regions
of sass_regions.py (prologue / term preamble / DFMA bodies / rest), each with
its stall-sample split, and the top instructions by `wait` and `dispatch`
stalls.  Usage: python scripts/sass_stalls.py gpurun_out/ncu_sass_qd.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie = h.index("Instructions Executed")
body = rows[2:]
n = [int(r[ie] or 0) for r in body]
top = max(n)
dfma = [i for i, r in enumerate(body) if r[1].strip().startswith("DFMA") and n[i] >= top * 0.6]
first_hot = next(i for i in range(len(body)) if n[i] >= top * 0.6)
regions = {"prologue": (0, first_hot), "term_pre": (first_hot, dfma[0]), "bodies": (dfma[0], dfma[-1] + 1),
           "rest": (dfma[-1] + 1, len(body))}
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in cols}
tot = sum(int(r[idx[c]] or 0) for r in body for c in cols) or 1
for k, (a, b) in regions.items():
    st = collections.Counter()
    for r in body[a:b]:
        for c in cols:
            st[c[6:]] += int(r[idx[c]] or 0)
    s = sum(st.values())
    print(f"{k:9s} {100 * s / tot:5.1f}% of samples:", {c: round(100 * v / tot, 1) for c, v in st.most_common(6)})
for c in ("stall_wait", "stall_dispatch"):
    best = sorted(range(len(body)), key=lambda i: -int(body[i][idx[c]] or 0))[:8]
    print(c, [(i, body[i][1].strip()[:40], body[i][idx[c]]) for i in best])

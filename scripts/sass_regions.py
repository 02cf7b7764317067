"""Region breakdown of an ncu source-page (SASS) CSV: stall samples and
instruction counts in prologue / term preamble / DFMA bodies / rest, plus the
opcode mix.  Usage: python scripts/sass_regions.py gpurun_out/ncu_sass_od.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
body = rows[2:]
n = [int(r[ie] or 0) for r in body]
top = max(n)
dfma = [i for i, r in enumerate(body) if r[1].strip().startswith("DFMA") and n[i] >= top * 0.6]
T = sum(int(r[ss] or 0) for r in body)
tot = sum(n)
print("hot DFMA lines", len(dfma), dfma[0], dfma[-1])
first_hot = next(i for i in range(len(body)) if n[i] >= top * 0.6)
regions = {"prologue": (0, first_hot), "term_pre": (first_hot, dfma[0]), "bodies": (dfma[0], dfma[-1] + 1),
           "rest": (dfma[-1] + 1, len(body))}
for k, (a, b) in regions.items():
    s = sum(int(r[ss] or 0) for r in body[a:b])
    print(f"{k:10s} samples {100 * s / T:5.1f}%  inst {100 * sum(n[a:b]) / tot:5.1f}%")
cnt = collections.Counter()
for r, c in zip(body, n):
    op = r[1].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    cnt[o.split(".")[0]] += c
print({k: round(100 * v / tot, 2) for k, v in cnt.most_common(12)}, "total warp inst", tot)

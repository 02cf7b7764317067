"""Region breakdown of an ncu source-page (SASS) CSV: stall samples and
instruction counts in the DFMA bodies (runs of hot DFMA lines, one per code
copy: the kernel has one per part), the per-term code around them (other
lines executed about as often), the prologue (cold lines before the first
body) and the rest (cold lines after: epilogue), plus the opcode mix and the
stall reasons per region.  Usage: python scripts/sass_regions.py sass.csv"""
import collections
import csv
import sys


def regions(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    body = rows[2:]
    n = [int(r[ie] or 0) for r in body]
    top = max(n)
    hot = [i for i in range(len(body)) if n[i] >= 0.3 * top]
    dfma = [i for i in hot if body[i][1].strip().startswith("DFMA")]
    runs, start, prev = [], dfma[0], dfma[0]
    for i in dfma[1:]:
        if i - prev > 40:
            runs.append((start, prev))
            start = i
        prev = i
    runs.append((start, prev))
    runs = [r for r in runs if r[1] - r[0] > 20]
    inbody = set()
    for a, b in runs:
        inbody.update(range(a, b + 1))
    first = runs[0][0]
    reg = {}
    for i in range(len(body)):
        if i in inbody:
            reg[i] = "bodies"
        elif n[i] >= 0.3 * top:
            reg[i] = "term_code"
        elif i < first:
            reg[i] = "prologue"
        else:
            reg[i] = "rest"
    return body, h, n, reg, runs


if __name__ == "__main__":
    body, h, n, reg, runs = regions(sys.argv[1])
    ss = h.index("Warp Stall Sampling (All Samples)")
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    idx = {c: h.index(c) for c in cols}
    T = sum(int(r[ss] or 0) for r in body) or 1
    tot = sum(n)
    print("DFMA bodies (line ranges):", runs)
    for name in ("prologue", "term_code", "bodies", "rest"):
        ids = [i for i in reg if reg[i] == name]
        s = sum(int(body[i][ss] or 0) for i in ids)
        st = collections.Counter()
        for i in ids:
            for c in cols:
                st[c[6:]] += int(body[i][idx[c]] or 0)
        print(f"{name:10s} samples {100 * s / T:5.1f}%  inst {100 * sum(n[i] for i in ids) / tot:5.1f}%  stalls",
              {c: round(100 * v / T, 1) for c, v in st.most_common(5)})
    cnt = collections.Counter()
    for r, c in zip(body, n):
        op = r[1].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        cnt[o.split(".")[0] + (".128" if ".128" in o else "")] += c
    print({k: round(100 * v / tot, 2) for k, v in cnt.most_common(12)}, "total warp inst", tot)

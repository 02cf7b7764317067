"""Opcode mix and hottest SASS lines of one kernel from `ncu --page source --print-source sass --csv`."""
import collections
import csv
import sys


def main(path, top=15):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if "Instructions Executed" in r and "Source" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0] != "Address":
            data.append(r)
    ia, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
    iw, ith = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Avg. Threads Executed")

    def f(x):
        try:
            return float(x.replace(",", "") or 0)
        except ValueError:
            return 0.0
    tot = sum(f(r[ia]) for r in data)
    totw = sum(f(r[iw]) for r in data) or 1
    print("warp instructions", tot, "stall samples", totw)
    op, opw, thr = collections.Counter(), collections.Counter(), collections.defaultdict(float)
    for r in data:
        t = r[isrc].split()
        if not t:
            continue
        o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        op[o] += f(r[ia])
        opw[o] += f(r[iw])
        thr[o] += f(r[ia]) * f(r[ith])
    for o, c in op.most_common(22):
        print(f"{o:10s} {c / tot * 100:6.2f}% inst {opw[o] / totw * 100:6.2f}% samples  threads {thr[o] / max(c, 1):.1f}")
    for r in sorted(data, key=lambda r: -f(r[iw]))[:top]:
        print(r[0], r[isrc][:70], f(r[iw]), f(r[ia]))


if __name__ == "__main__":
    main(sys.argv[1])

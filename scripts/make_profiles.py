"""Copy the ncu evidence judged this round into profiles/ (tracked):
launch lists (per-kernel share of the bench step) and ncu --set full summaries."""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from ncu_summary import summarise  # noqa: E402


def launch_summary(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iv, iu, im = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name"))
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("void ", "")
        tot[name] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        cnt[name] += 1
    ours = {k: v for k, v in tot.items() if "mdps::" in k}
    s = sum(ours.values())
    return [{"kernel": k, "launches": cnt[k], "ms_total": round(v, 4), "share_of_mdps_time": round(v / s, 4)}
            for k, v in sorted(ours.items(), key=lambda kv: -kv[1])]


if __name__ == "__main__":
    tag = sys.argv[1]
    out = {}
    for arg in sys.argv[2:]:
        kind, path = arg.split("=", 1)
        if kind == "launches":
            out.setdefault("launch_lists", {})[os.path.basename(path)] = launch_summary(path)
        else:
            out.setdefault("ncu_full", {})[os.path.basename(path)] = summarise(path)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    dst = os.path.join(ROOT, "profiles", f"{tag}.json")
    json.dump(out, open(dst, "w"), indent=1)
    print(dst)

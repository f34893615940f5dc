"""Stall reasons by CUDA source line from an ncu source page
(--page source --csv --print-source cuda,sass, optionally gzipped).
Usage: python profiles/stallagg.py src.csv[.gz] [topN]"""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
rows = list(csv.reader(f))
hdr, cur = None, None
agg = collections.defaultdict(lambda: collections.Counter())
srcs = {}
tot = collections.Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        idx = {h: i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
        continue
    if hdr is None or not r[0].isdigit():
        continue
    key = (cur, int(r[0]))
    srcs[key] = r[1][:70]
    for h, i in idx.items():
        try:
            v = int(r[i])
        except (ValueError, IndexError):
            continue
        agg[key][h] += v
        tot[h] += v
T = sum(tot.values())
print("overall:", ", ".join(f"{h[6:]} {100*v/T:.1f}%" for h, v in tot.most_common(10)))
for key, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    s = sum(c.values())
    reasons = ", ".join(f"{h[6:]} {100*v/s:.0f}" for h, v in c.most_common(3))
    print(f"{100*s/T:5.1f}%  {key[0]}:{key[1]:<5d} [{reasons}]  {srcs[key]}")

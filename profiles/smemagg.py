"""Aggregate an ncu source page (--print-source cuda,sass --csv) by CUDA source
line: shared-memory wavefronts, excess (bank-conflict) wavefronts, stall samples.
Usage: python profiles/smemagg.py src.csv[.gz] [topN]"""
import collections, csv, gzip, sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fh = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
agg = collections.defaultdict(lambda: [0, 0, 0, ""])
hdr = None
cur = None
for r in csv.reader(fh):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or not r[0].isdigit():
        continue
    def num(k):
        try:
            return int(float(r[hdr[k]].replace(",", "")))
        except (ValueError, KeyError, IndexError):
            return 0
    a = agg[(cur, int(r[0]))]
    a[0] += num("L1 Wavefronts Shared")
    a[1] += num("L1 Wavefronts Shared Excessive")
    a[2] += num("Warp Stall Sampling (All Samples)")
    a[3] = r[1][:80]
tw = sum(v[0] for v in agg.values()) or 1
te = sum(v[1] for v in agg.values())
ts = sum(v[2] for v in agg.values()) or 1
print(f"shared wavefronts {tw}, excessive {te} ({100*te/tw:.1f}%), samples {ts}")
print("  wavef%  excess%  stall%  line")
for (f, ln), (w, e, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"  {100*w/tw:5.1f}  {100*e/tw:6.1f}  {100*s/ts:6.1f}  {f}:{ln} {src}")

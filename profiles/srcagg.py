"""Aggregate an ncu source page (--print-source cuda,sass --csv) by CUDA source
line: warp-stall samples and executed instructions.  Usage:
  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
  python profiles/srcagg.py src.csv [topN]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
files = {}
agg = collections.defaultdict(lambda: [0, 0, ""])
cur_file = None
hdr = None
total = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] not in ("", "-") and r[0].isdigit():
        key = (cur_file, int(r[0]))
        try:
            s = int(r[4]); ins = int(r[7])
        except ValueError:
            continue
        agg[key][0] += s
        agg[key][1] += ins
        agg[key][2] = r[1][:90]
        total += s
print(f"total samples {total}")
for (f, ln), (s, ins, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/total:5.1f}%  {ins:>11d}  {f}:{ln:<5d} {src}")

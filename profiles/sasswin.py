"""SASS in address order with warp-stall samples and source line, from an ncu
source page (--print-source cuda,sass --csv[.gz]).  Prints the windows around
the N instructions with the most samples.
Usage: python profiles/sasswin.py src.csv[.gz] [N] [window]"""
import csv
import gzip
import sys

path = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
W = int(sys.argv[3]) if len(sys.argv) > 3 else 6
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
cur, line, src = None, None, ""
ins = []
for r in csv.reader(f):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        continue
    if r[0].isdigit():
        line, src = int(r[0]), r[1][:60]
        continue
    if len(r) > 4 and r[2].startswith("0x"):
        try:
            ins.append((int(r[2], 16), r[3].strip(), int(r[4]), f"{cur}:{line}", src))
        except ValueError:
            pass
ins.sort()
tot = sum(i[2] for i in ins)
hot = sorted(range(len(ins)), key=lambda k: -ins[k][2])[:N]
shown = set()
for h in sorted(hot):
    print("-" * 100)
    for k in range(max(0, h - W), min(len(ins), h + 3)):
        if k in shown:
            continue
        shown.add(k)
        a, s, n, loc, src = ins[k]
        mark = ">>" if k == h else "  "
        print(f"{mark}{100*n/tot:5.1f}% {a & 0xfffff:6x} {s[:60]:60s} {loc}")

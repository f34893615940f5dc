"""Record per-launch DRAM traffic of the solve kernel from `ncu --set full`
raw CSV exports (exp/ncu_cap.sh) into profiles/ncu_traffic.json, which
bench.py reads for roofline.traffic.  Usage:
  python profiles/make_traffic.py WORKLOAD RAW_CSV REALIZATIONS_IN_CAPTURE [round]"""
import csv
import json
import os
import sys

name, path, nreal = sys.argv[1], sys.argv[2], int(sys.argv[3])
rnd = sys.argv[4] if len(sys.argv) > 4 else "r01"
rows = list(csv.reader(open(path)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def nbytes(key):
    return float(d[key].replace(",", "")) * scale[u[key]]


rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
dur = float(d["gpu__time_duration.sum"].replace(",", ""))
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
db = json.load(open(out)) if os.path.exists(out) else {}
db[name] = {"dram_read_bytes": rd, "dram_write_bytes": wr, "realizations": nreal,
            "bytes_per_realization": (rd + wr) / nreal,
            "duration": f"{dur} {u['gpu__time_duration.sum']}",
            "kernel": d.get("Kernel Name", ""), "source": f"profiles/{rnd}_ncu_{name}.md"}
json.dump(db, open(out, "w"), indent=1, sort_keys=True)
print(name, db[name])

"""Markdown summary of one `ncu --set full` capture exported by exp/ncu_cap.sh
(details / raw / source CSVs).  Usage:
  python profiles/ncu_summary.py NAME GPURUN_DIR "command line" > profiles/r01_ncu_NAME.md"""
import csv
import gzip
import os
import subprocess
import sys

name, d, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
raw = list(csv.reader(open(os.path.join(d, f"ncu_{name}_raw.csv"))))
R = dict(zip(raw[0], raw[2]))
U = dict(zip(raw[0], raw[1]))


def m(key, fmt="{}"):
    v = R.get(key, "n/a")
    return fmt.format(v) + (" " + U[key] if U.get(key) else "")


print(f"# ncu --set full: `{R.get('Kernel Name', '?')}` ({name})\n")
print(f"Command: `{cmd}`  \nCapture: `ncu --set full --clock-control none --import-source on -c 1` "
      f"(exp/ncu_cap.sh); numbers read with `ncu -i ... --page raw|details|source --csv`.\n")
rows = [
    ("duration", "gpu__time_duration.sum"),
    ("grid x block", None),
    ("registers / thread", "launch__registers_per_thread"),
    ("dynamic shared memory / block", "launch__shared_mem_per_block_dynamic"),
    ("achieved occupancy (warps)", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("issue slots busy", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("FMA pipe (fp32) active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("FP64 pipe active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("shared-memory wavefronts / peak", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    ("shared bank conflicts (excess wavefronts)", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM throughput / peak", "dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("L2 hit rate", "lts__t_sector_hit_rate.pct"),
]
print("| metric | value |\n|---|---|")
for label, key in rows:
    if key is None:
        print(f"| {label} | {R.get('launch__grid_size', '?')} x {R.get('launch__block_size', '?')} "
              f"(cluster {R.get('launch__cluster_dim_x', '1')}) |")
    else:
        print(f"| {label} | {m(key)} |")
items = []
for h, v in R.items():
    if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
        try:
            items.append((float(v.replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError:
            pass
tot = sum(x for x, _ in items) or 1
print("\nWarp-state samples: " + ", ".join(f"{k} {100 * x / tot:.1f}%" for x, k in sorted(items, reverse=True)[:10]))
here = os.path.dirname(os.path.abspath(__file__))
src = os.path.join(d, f"ncu_{name}_src.csv.gz")
print("\nStall samples by source line (profiles/srcagg.py, top 25):\n\n```")
tmp = "/tmp/_src.csv"
with gzip.open(src, "rt") as f, open(tmp, "w") as g:
    g.write(f.read())
print(subprocess.run([sys.executable, os.path.join(here, "srcagg.py"), tmp, "25"], capture_output=True,
                     text=True).stdout.rstrip())
print("```\n\nShared-memory wavefronts by source line (profiles/smemagg.py, top 12):\n\n```")
print(subprocess.run([sys.executable, os.path.join(here, "smemagg.py"), src, "12"], capture_output=True,
                     text=True).stdout.rstrip())
print("```")

"""Print a table of bench_<cfg>.json lines (gpurun_out/ or a given dir)."""
import glob, json, os, sys
d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
print(f"| workload | realizations/GPU-step | mean iters | value (real./s) | e2e (real./s) | ms/step | kernel TFLOP/s (F-basis) | frac of FFMA peak | BCGD-step share | BCGD-step frac | CPU port (real./s, cores) | GPU/CPU |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for f in sorted(glob.glob(os.path.join(d, "bench_*.json"))):
    try:
        dd = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    c, r, cb, e = dd["config"], dd["roofline"], dd.get("cpu_baseline") or {}, dd.get("e2e") or {}
    ratio = dd["value"] / cb["value"] if cb.get("value") else float("nan")
    print(f"| {c['workload']} | {c['realizations_per_gpu_step']} | {c['mean_iterations']:.1f} | {dd['value']:.1f} | "
          f"{e.get('value', float('nan')):.1f} | {dd['ms_per_step']:.1f} | {r['achieved']:.2f} | {r['frac']:.3f} | "
          f"{(r.get('bcgd_step') or {}).get('share_of_kernel', float('nan')):.3f} | {(r.get('bcgd_step') or {}).get('frac', float('nan')):.3f} | "
          f"{cb.get('value', float('nan')):.3f} ({cb.get('cores')}) | {ratio:.0f}x |")

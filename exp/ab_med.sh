# A/B of engine builds on the single-CTA workloads: bash exp/ab_med.sh lib1 lib2 ...
for lib in "$@"; do
  for cfg in "medium" "sweep64 --per-block 16384" "sweep32 --per-block 16384"; do
    set -- $cfg
    AMMMSE_LIB=$lib timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abm.json 2> gpurun_out/abm.err
    echo "$lib $1 $(python -c "import json;d=json.load(open('gpurun_out/abm.json'));print(round(d['value'],1), round(d['roofline']['frac'],3))")"
  done
done

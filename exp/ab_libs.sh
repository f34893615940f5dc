# A/B of engine builds: bash exp/ab_libs.sh lib1 lib2 ...
for lib in "$@"; do
  for cfg in "large --per-block 1024" "massive --per-block 2048" "sweep128 --per-block 8192" "sweep256 --per-block 4096"; do
    set -- $cfg
    AMMMSE_LIB=$lib timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/abl.json 2> gpurun_out/abl.err
    echo "$lib $1 $(python -c "import json;d=json.load(open('gpurun_out/abl.json'));print(round(d['value'],1), round(d['roofline']['frac'],3))")"
  done
done

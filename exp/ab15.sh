timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_v15.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_v15.log; grep -E "^FAILED" gpurun_out/pytest_v15.log | head -8
for ns in 1 0; do
  for cfg in "large --per-block 1024" "massive --per-block 2048" "sweep128 --per-block 8192" "sweep256 --per-block 4096" "sweep512 --per-block 1024"; do
    set -- $cfg
    AMMMSE_NO_SPEC=$ns timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-phase-profile > gpurun_out/abl.json 2> gpurun_out/abl.err
    echo "no_spec=$ns $1 $(python -c "import json;d=json.load(open('gpurun_out/abl.json'));print(round(d['value'],1), round(d['roofline']['frac'],3))")"
  done
done

timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_v16.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_v16.log; grep -E "^FAILED" gpurun_out/pytest_v16.log | head -8
for ns in 1 0; do
  for cfg in "small" "sweep32 --per-block 16384" "medium"; do
    set -- $cfg
    AMMMSE_NO_SPEC=$ns timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-phase-profile > gpurun_out/abl.json 2> gpurun_out/abl.err
    echo "no_spec=$ns $1 $(python -c "import json;d=json.load(open('gpurun_out/abl.json'));print(round(d['value'],1), round(d['roofline']['frac'],3))")"
  done
done

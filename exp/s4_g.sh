export PATH=/usr/local/cuda/bin:$PATH
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s4_full_tests.log 2>&1; tail -5 gpurun_out/s4_full_tests.log
timeout 900 python bench.py > gpurun_out/s4_bench_default.json 2> gpurun_out/s4_bench_default.err; tail -c 300 gpurun_out/s4_bench_default.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/s4_bench_default.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e'], d['config']['engine'], d['parity'], d['roofline']['frac'], d['cpu_baseline']['value'])
PY

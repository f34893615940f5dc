export PATH=/usr/local/cuda/bin:$PATH
timeout 1800 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/s4_full_tests.log 2>&1; tail -14 gpurun_out/s4_full_tests.log
timeout 600 python bench.py --per-block 2048 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/s4_prod.json 2> gpurun_out/s4_prod.err; tail -c 200 gpurun_out/s4_prod.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/s4_prod.json').read().strip().splitlines()[-1])
print('prod lib:', d['value'], d['config']['mean_iterations'], d['config']['failed_realizations'], d['config']['engine'])
PY

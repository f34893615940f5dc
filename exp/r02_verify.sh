export PATH=/usr/local/cuda/bin:$PATH
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/last_tests.log 2>&1; tail -2 gpurun_out/last_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/last_bench.json 2> gpurun_out/last_bench.err; tail -c 200 gpurun_out/last_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/last_bench.json').read().strip().splitlines()[-1])
print('default:', d['value'], d['e2e']['value'], d['parity']['wsr_rel_max'], d['parity']['iterations_mismatch'], d['roofline']['frac'])
PY

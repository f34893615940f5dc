timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_c5.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_c5.log; grep -E "^FAILED|^E  " gpurun_out/pytest_c5.log | head -12
timeout 600 python bench.py --config small --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err; echo "small rc=$? $(python -c "import json;d=json.load(open('gpurun_out/bench_small.json'));print(round(d['value']), round(d['e2e']['value']))")"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1

export PATH=/usr/local/cuda/bin:$PATH
export PYTHONPATH=$PWD
export AMMMSE_LIB=paper_2510_20507_b200/libammmse_dev.so
timeout 900 python -m pytest tests/test_gpu_tc2.py tests/test_gpu_golden.py -k "(tc2 or large) and not planner" -x -q > gpurun_out/s4_tc2_tests.log 2>&1; tail -3 gpurun_out/s4_tc2_tests.log
timeout 200 python exp/s4_tc2.py 16 2>&1 | grep -E "residual|deferred" | head -4
for sp in 0 0; do
timeout 600 python bench.py --per-block 2048 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/s4_f_$sp.json 2> gpurun_out/s4_f_$sp.err
python - <<PY
import json
d=json.loads(open('gpurun_out/s4_f_$sp.json').read().strip().splitlines()[-1])
print('dev:', d['value'], d['config']['mean_iterations'], d['config']['failed_realizations'])
PY
done

export PATH=/usr/local/cuda/bin:$PATH
for sp in 1 0 1; do
AMMMSE_TC2_WSR_SPLIT=$sp timeout 600 python bench.py --per-block 2048 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/s4_i_$sp.json 2> gpurun_out/s4_i_$sp.err
python - <<PY
import json
d=json.loads(open('gpurun_out/s4_i_$sp.json').read().strip().splitlines()[-1])
print('prod split $sp:', d['value'], d['config']['mean_iterations'], d['config']['failed_realizations'], d['clocks']['sm_mhz'])
PY
done

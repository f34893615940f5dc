export PATH=/usr/local/cuda/bin:$PATH
export PYTHONPATH=$PWD
export AMMMSE_LIB=paper_2510_20507_b200/libammmse_dev.so
timeout 300 python -m pytest tests/test_gpu_golden.py -k "large" -x -q -s > gpurun_out/s4_tc2_golden.log 2>&1; tail -5 gpurun_out/s4_tc2_golden.log
for dbg in 0; do
AMMMSE_DBG=$dbg timeout 600 python bench.py --per-block 512 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --phase-profile > gpurun_out/s4_tc2_phase_$dbg.json 2> gpurun_out/s4_tc2_phase_$dbg.err; tail -c 300 gpurun_out/s4_tc2_phase_$dbg.err
python - <<PY
import json
d=json.loads(open('gpurun_out/s4_tc2_phase_$dbg.json').read().strip().splitlines()[-1])
v=d['value']; it=d['config']['mean_iterations']
cyc=1965e6*33/(v*it)
print('dbg $dbg', v, it, 'cycles/iter', cyc, d['config']['failed_realizations'])
print([round(x*cyc) for x in d['roofline'].get('bcgd_step',{}).get('phases')])
PY
done

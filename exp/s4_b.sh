export PATH=/usr/local/cuda/bin:$PATH
export PYTHONPATH=$PWD
export AMMMSE_LIB=paper_2510_20507_b200/libammmse_dev.so
for dbg in 0; do
AMMMSE_DBG=$dbg timeout 600 python bench.py --per-block 512 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --phase-profile > gpurun_out/s4_tc2_phase_$dbg.json 2> gpurun_out/s4_tc2_phase_$dbg.err; tail -c 300 gpurun_out/s4_tc2_phase_$dbg.err
python - <<PY
import json
d=json.loads(open('gpurun_out/s4_tc2_phase_$dbg.json').read().strip().splitlines()[-1])
v=d['value']; it=d['config']['mean_iterations']
cyc=1965e6*33/(v*it)
ph=d['roofline'].get('bcgd_step',{}).get('phases')
tot=sum(ph[:17])
print('dbg $dbg', v, it, 'cycles/iter', cyc, d['config']['failed_realizations'])
tot=sum(ph[:19])
print([round(x/tot*cyc) for x in ph[:19]], 'producer-0 done-wait per iter (CTA 0, x132):', round(ph[19]/tot*cyc*132))
PY
done

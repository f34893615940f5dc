export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; tail -3 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -c 300 gpurun_out/final_bench.err
for tc in 1 2 3; do
timeout 600 python bench.py --per-block 2048 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --tensor-cores $tc > gpurun_out/final_ab_large_$tc.json 2> gpurun_out/final_ab_large_$tc.err
done
python - <<'PY'
import json
d=json.loads(open('gpurun_out/final_bench.json').read().strip().splitlines()[-1])
print('default:', d['value'], d['e2e']['value'], d['parity']['wsr_rel_max'], d['parity']['iterations_mismatch'], d['roofline']['frac'], d['cpu_baseline']['value'])
for tc in (1,2,3):
    x=json.loads(open(f'gpurun_out/final_ab_large_{tc}.json').read().strip().splitlines()[-1])
    print('tensor_cores', tc, x['value'], x['config']['engine']['tensor_cores'])
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --per-block 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --gen-workers 1 > gpurun_out/final_ncu_launches.log 2>&1; grep -c ammmse gpurun_out/final_launches.csv
bash exp/ncu_cap.sh tc2final ammmse_tc2 --per-block 132
python profiles/stallagg.py gpurun_out/ncu_tc2final_src.csv.gz 40 > gpurun_out/ncu_tc2final_stalls.txt 2>&1; head -12 gpurun_out/ncu_tc2final_stalls.txt

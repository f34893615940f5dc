export PATH=/usr/local/cuda/bin:$PATH
export PYTHONPATH=$PWD
export AMMMSE_LIB=paper_2510_20507_b200/libammmse_dev.so
for d in 1 0; do
AMMMSE_TC2_DEFER=$d timeout 600 python bench.py --per-block 2048 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/s4_f_$d.json 2> gpurun_out/s4_f_$d.err; tail -c 200 gpurun_out/s4_f_$d.err
python - <<PY
import json
d=json.loads(open('gpurun_out/s4_f_$d.json').read().strip().splitlines()[-1])
print('defer $d', d['value'], d['config']['mean_iterations'], d['config']['failed_realizations'])
PY
done
bash exp/ncu_cap.sh tc2 ammmse_tc2 --per-block 132
python profiles/stallagg.py gpurun_out/ncu_tc2_src.csv.gz 45 > gpurun_out/ncu_tc2_stalls.txt 2>&1; head -50 gpurun_out/ncu_tc2_stalls.txt

# phase timers for the cluster workloads + ncu launch list + ncu --set full captures
mkdir -p gpurun_out
ph() { name=$1; shift; AMMMSE_PROFILE_PHASES=1 timeout 600 python bench.py --config $name --steps 1 --warmup 1 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ph_$name.json 2> gpurun_out/ph_$name.err; echo "$name rc=$?"; grep -i phase gpurun_out/ph_$name.err | tail -3; python -c "import json;d=json.load(open('gpurun_out/ph_$name.json'));print(d['value'], d['roofline']['frac'])"; }
ph massive --per-block 1024
ph large --per-block 512
ph sweep128 --per-block 4096
ph sweep256 --per-block 1024
ph medium --per-block 1024
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_medium.csv python bench.py --steps 1 --warmup 1 --per-block 256 --no-e2e --no-cpu-baseline --gen-workers 1 > gpurun_out/ncu_ll.log 2>&1; echo "ll rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ammmse_solve -c 1 -o gpurun_out/prof_medium -f python bench.py --steps 1 --warmup 0 --per-block 256 --no-e2e --no-cpu-baseline --gen-workers 1 > gpurun_out/ncu_med.log 2>&1; echo "ncu med rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ammmse_cluster -c 1 -o gpurun_out/prof_massive -f python bench.py --config massive --steps 1 --warmup 0 --per-block 64 --no-e2e --no-cpu-baseline --gen-workers 1 > gpurun_out/ncu_mas.log 2>&1; echo "ncu massive rc=$?"
ls -la gpurun_out

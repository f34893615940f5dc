ph() { name=$1; shift; AMMMSE_PROFILE_PHASES=1 timeout 600 python bench.py --config $name --steps 1 --warmup 1 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ph_$name.json 2> gpurun_out/ph_$name.err; echo "$name rc=$?"; grep -i phase gpurun_out/ph_$name.err | tail -1; }
ph medium --per-block 1024
ph large --per-block 512
ph massive --per-block 1024
ph sweep128 --per-block 4096
bash exp/ncu_cap.sh medium ammmse_solve --per-block 256
bash exp/ncu_cap.sh massive ammmse_cluster --config massive --per-block 256
bash exp/ncu_cap.sh sweep128 ammmse_cluster --config sweep128 --per-block 1024

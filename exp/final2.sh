nproc
bash profiles/bench_all.sh
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 1 --warmup 1 --per-block 256 --no-e2e --no-cpu-baseline --no-phase-profile --gen-workers 1 > gpurun_out/ncu_ll.log 2>&1; echo "ll rc=$?"
bash exp/ncu_cap.sh medium ammmse_solve --per-block 256 --no-phase-profile
bash exp/ncu_cap.sh massive ammmse_cluster --config massive --per-block 256 --no-phase-profile
bash exp/ncu_cap.sh sweep128 ammmse_cluster --config sweep128 --per-block 1024 --no-phase-profile
bash exp/ncu_cap.sh large ammmse_cluster --config large --per-block 128 --no-phase-profile

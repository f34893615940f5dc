export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/t18.log 2>&1; tail -5 gpurun_out/t18.log
python bench.py --steps 2 --warmup 1 > gpurun_out/b18.log 2>&1; tail -c 5000 gpurun_out/b18.log
python bench.py --per-block 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --gen-workers 4 > gpurun_out/plain18.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 8 --csv --log-file gpurun_out/r02_launches.csv python bench.py --per-block 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --gen-workers 4 > gpurun_out/ncu18.log 2>&1
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --gen-workers 1 --per-block 132 > gpurun_out/plain18b.log 2>&1 && bash exp/ncu_cap.sh large_tc2 cluster_kernel --per-block 132

export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t23.log 2>&1; tail -4 gpurun_out/t23.log
python bench.py --steps 3 --warmup 2 > gpurun_out/b23.log 2>&1; tail -c 1800 gpurun_out/b23.log
python bench_gemmstep.py > gpurun_out/gemmstep23.jsonl 2>&1
bash exp/ab_tc.sh
python bench.py --per-block 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --gen-workers 4 > gpurun_out/plain23.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 8 --csv --log-file gpurun_out/r02_launches.csv python bench.py --per-block 512 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --gen-workers 4 > gpurun_out/ncu23.log 2>&1
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --gen-workers 1 --per-block 132 > gpurun_out/plain23b.log 2>&1 && bash exp/ncu_cap.sh large_tc3 cluster_kernel --per-block 132

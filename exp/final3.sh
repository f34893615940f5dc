timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_f3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_f3.log; grep -E "^FAILED" gpurun_out/pytest_f3.log | head -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_medium.json 2> gpurun_out/bench_medium.err; echo "bench rc=$?"; cat gpurun_out/bench_medium.json | head -c 400; echo
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 1 --warmup 1 --per-block 256 --no-e2e --no-cpu-baseline --no-phase-profile --gen-workers 1 > gpurun_out/ncu_ll.log 2>&1; echo "ll rc=$?"
bash exp/ncu_cap.sh medium ammmse_solve --per-block 256 --no-phase-profile

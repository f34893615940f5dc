for lib in build/ab/v4.so build/ab/v7.so; do echo "== $lib"; AMMMSE_LIB=$lib timeout 600 python exp/rel_dev.py 2>&1 | tail -30; done
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_v7.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_v7.log; grep -E "^FAILED" gpurun_out/pytest_v7.log | head -8
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_v7.json 2> gpurun_out/bench_v7.err; echo "bench rc=$?"; cat gpurun_out/bench_v7.json

export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4_tests.log 2>&1; tail -3 gpurun_out/s4_tests.log
AMMMSE_LIB=paper_2510_20507_b200/libammmse_phases.so timeout 600 python bench.py --per-block 1024 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --phase-profile > gpurun_out/s4_phase_large.json 2> gpurun_out/s4_phase_large.err; tail -c 1500 gpurun_out/s4_phase_large.json
AMMMSE_LIB=paper_2510_20507_b200/libammmse_phases.so timeout 600 python bench.py --per-block 1024 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --phase-profile --tensor-cores 2 > gpurun_out/s4_phase_large_ffma.json 2> gpurun_out/s4_phase_large_ffma.err

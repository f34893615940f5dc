export PATH=/usr/local/cuda/bin:$PATH
export PYTHONPATH=$PWD
export AMMMSE_LIB=paper_2510_20507_b200/libammmse_dev.so
timeout 900 python -m pytest tests/test_gpu_tc2.py tests/test_gpu_golden.py -k "(tc2 or large) and not planner" -x -q > gpurun_out/s4_tc2_tests.log 2>&1; tail -4 gpurun_out/s4_tc2_tests.log

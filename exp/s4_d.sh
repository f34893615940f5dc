export PATH=/usr/local/cuda/bin:$PATH
export PYTHONPATH=$PWD
export AMMMSE_LIB=paper_2510_20507_b200/libammmse_dev.so
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python exp/s4_tc2.py 4 > gpurun_out/s4_sanitizer.log 2>&1; grep -v "^$" gpurun_out/s4_sanitizer.log | head -60

export PATH=/usr/local/cuda/bin:$PATH
export PYTHONPATH=$PWD
export AMMMSE_LIB=paper_2510_20507_b200/libammmse_dev.so
timeout 200 python exp/s4_tc2.py 64 2>&1 | tail -16

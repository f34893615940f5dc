export PATH=/usr/local/cuda/bin:$PATH
export PYTHONPATH=$PWD
export AMMMSE_LIB=paper_2510_20507_b200/libammmse_dev.so
AMMMSE_DBG=0 timeout 120 python exp/s4_tc2.py 8 2>&1 | grep -E "tc=3|iters|Error|error" | head -3

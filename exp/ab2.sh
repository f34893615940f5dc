bash exp/ab_med.sh build/ab/splitmajor.so build/ab/v2.so
bash exp/ab_libs.sh build/ab/splitmajor.so build/ab/v2.so
AMMMSE_LIB=build/ab/v2.so timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2

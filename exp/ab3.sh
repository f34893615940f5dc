timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v3.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_v3.log
bash exp/ab_libs.sh build/ab/v2.so build/ab/v3.so

timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_v5.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_v5.log; grep FAILED gpurun_out/pytest_v5.log | head
bash exp/ab_libs.sh build/ab/v4.so build/ab/v5.so

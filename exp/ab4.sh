timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_v4.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_v4.log; grep FAILED gpurun_out/pytest_v4.log | head
bash exp/ab_med.sh build/ab/v2.so build/ab/v4.so
bash exp/ab_libs.sh build/ab/v4.so

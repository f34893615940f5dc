timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_v10.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_v10.log; grep -E "^FAILED" gpurun_out/pytest_v10.log | head -8
bash exp/ab_med.sh build/ab/v9.so build/ab/v10.so
bash exp/ab_libs.sh build/ab/v9.so build/ab/v10.so

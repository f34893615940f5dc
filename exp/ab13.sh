timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_v13.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_v13.log; grep -E "^FAILED" gpurun_out/pytest_v13.log | head -8
bash exp/ab_libs.sh build/ab/v12.so build/ab/v13.so

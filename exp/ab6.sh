timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_v6.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_v6.log; grep -E "^FAILED|^E  " gpurun_out/pytest_v6.log | head -8
bash exp/ab_med.sh build/ab/v4.so build/ab/v6.so
bash exp/ab_libs.sh build/ab/v6.so

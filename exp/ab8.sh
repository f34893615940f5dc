timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_v8.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_v8.log; grep -E "^FAILED" gpurun_out/pytest_v8.log | head -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash exp/ab_libs.sh build/ab/v8.so

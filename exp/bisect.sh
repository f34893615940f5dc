for lib in build/ab/v4.so build/ab/var_A0.so build/ab/var_B0.so build/ab/var_AB0.so build/ab/v7.so; do
  AMMMSE_LIB=$lib timeout 600 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py -q -k "massive or sweep128 or sweep256 or large or cluster_engine_complex64 or odd_stage" > gpurun_out/bis.log 2>&1
  echo "$lib: $(tail -1 gpurun_out/bis.log)"
done

export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_gpu_integration.py tests/test_gpu_golden.py -q -k "integration or long or large" > gpurun_out/t24.log 2>&1; tail -4 gpurun_out/t24.log
python bench_gemmstep.py --reps 50 > gpurun_out/gs24.log 2>&1 && ncu --set full --clock-control none -k regex:gemm_step -s 2 -c 1 -o /tmp/gs python bench_gemmstep.py --reps 50 > gpurun_out/ncu_gs.log 2>&1; ncu -i /tmp/gs.ncu-rep --page raw --csv > gpurun_out/ncu_gemmstep_raw.csv 2>&1; ncu -i /tmp/gs.ncu-rep --page details --csv > gpurun_out/ncu_gemmstep_details.csv 2>&1

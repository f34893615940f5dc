# A/B of the cluster-engine GEMMs: FFMA (tensor_cores=2) vs tcgen05 (1) per workload
for spec in "large 2048" "massive 1024" "sweep128 8192" "sweep256 2048" "sweep512 256"; do
  set -- $spec
  for tc in 2 1; do
    timeout 400 python bench.py --config $1 --per-block $2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --tensor-cores $tc > gpurun_out/ab_$1_$tc.log 2>&1
    python -c "import json,sys;d=json.loads(open('gpurun_out/ab_$1_$tc.log').read().strip().splitlines()[-1]);print('$1', $tc, round(d['value'],1), d['config']['mean_iterations'], round(d['roofline']['frac'],3))" 2>/dev/null || (echo "$1 $tc FAILED"; tail -3 gpurun_out/ab_$1_$tc.log)
  done
done

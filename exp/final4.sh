run() { name=$1; tag=$2; shift 2; timeout 1200 python bench.py --config $name "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "$tag rc=$?"; grep "ammmse phases" gpurun_out/bench_$tag.err | tail -1; }
run large large --steps 3 --warmup 3 --cpu-seconds 20
run massive massive --steps 3 --warmup 3 --per-block 4096 --cpu-seconds 20 --no-e2e
run sweep128 sweep128 --steps 3 --warmup 3 --per-block 16384 --cpu-seconds 10 --no-e2e
run sweep256 sweep256 --steps 3 --warmup 3 --per-block 16384 --cpu-seconds 10 --no-e2e
run sweep512 sweep512 --steps 3 --warmup 3 --per-block 2048 --cpu-seconds 30 --no-e2e
run massive massive_device_B16384 --device-inputs --steps 3 --warmup 3 --cpu-seconds 10
run sweep128 sweep128_device_B65536 --device-inputs --steps 3 --warmup 3 --cpu-seconds 5
run sweep256 sweep256_device_B65536 --device-inputs --steps 3 --warmup 3 --cpu-seconds 5
bash exp/ncu_cap.sh massive ammmse_cluster --config massive --per-block 256 --no-phase-profile
bash exp/ncu_cap.sh sweep128 ammmse_cluster --config sweep128 --per-block 1024 --no-phase-profile
bash exp/ncu_cap.sh large ammmse_cluster --config large --per-block 128 --no-phase-profile

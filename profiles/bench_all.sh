#!/bin/bash
# Bench every BASELINE workload once (round summaries in profiles/); writes gpurun_out/bench_<cfg>.json
mkdir -p gpurun_out
run() { name=$1; tag=$2; shift 2; timeout 1200 python bench.py --config $name "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "$tag rc=$?"; grep "ammmse phases" gpurun_out/bench_$tag.err | tail -1; }
nproc
run medium medium --steps 3 --warmup 3 --cpu-seconds 20
run small small --steps 5 --warmup 3 --cpu-seconds 10
run large large --steps 3 --warmup 3 --cpu-seconds 20
run massive massive --steps 3 --warmup 3 --per-block 4096 --cpu-seconds 20 --no-e2e
for M in 32 64 128 256; do run sweep$M sweep$M --steps 3 --warmup 3 --per-block 16384 --cpu-seconds 10 --no-e2e; done
run sweep512 sweep512 --steps 3 --warmup 3 --per-block 2048 --cpu-seconds 30 --no-e2e
# full BASELINE batch sizes with on-device inputs (sweep512's 65536 would need 192 GB)
run massive massive_device_B16384 --device-inputs --steps 3 --warmup 3 --cpu-seconds 10
for M in 32 64 128 256; do run sweep$M sweep${M}_device_B65536 --device-inputs --steps 3 --warmup 3 --cpu-seconds 5; done

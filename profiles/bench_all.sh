#!/bin/bash
# Bench every BASELINE workload once (round summaries in profiles/); writes gpurun_out/bench_<cfg>.json
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 python bench.py --config $name "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err; echo "$name rc=$?"; tail -1 gpurun_out/bench_$name.err; }
nproc
run medium --steps 3 --warmup 3 --cpu-seconds 20
run small --steps 5 --warmup 3 --cpu-seconds 10
run large --steps 3 --warmup 3 --cpu-seconds 20
run massive --steps 3 --warmup 3 --per-block 4096 --cpu-seconds 20 --no-e2e
for M in 32 64 128 256; do run sweep$M --steps 3 --warmup 3 --per-block 16384 --cpu-seconds 10 --no-e2e; done
run sweep512 --steps 3 --warmup 3 --per-block 2048 --cpu-seconds 30 --no-e2e

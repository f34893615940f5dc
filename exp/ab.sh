python -m pytest tests -m gpu -x -q 2>&1 | tail -3
run() { name=$1; shift; timeout 900 python bench.py --config $name "$@" --no-cpu-baseline > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err; echo "$name rc=$? $(python -c "import json;d=json.load(open('gpurun_out/ab_$name.json'));print(d['value'], d['roofline']['frac'])")"; }
run medium --steps 3 --warmup 3
run massive --steps 3 --warmup 3 --per-block 2048 --no-e2e
run large --steps 3 --warmup 3 --per-block 1024 --no-e2e
run sweep128 --steps 3 --warmup 3 --per-block 8192 --no-e2e
run sweep256 --steps 3 --warmup 3 --per-block 4096 --no-e2e

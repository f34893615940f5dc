# quick GPU check: tests (bounded) + medium/small bench
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for cfg in "medium" "small"; do
  timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/q.json 2> gpurun_out/q.err
  echo "$cfg rc=$? $(python -c "import json;d=json.load(open('gpurun_out/q.json'));print(round(d['value'],1), round(d['roofline']['frac'],3), d['e2e']['value'] if d.get('e2e') else None)")"
done

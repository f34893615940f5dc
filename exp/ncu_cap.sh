# ncu --set full of one launch, exported to text on the box (reps are too large to ship back)
# usage: ncu_cap.sh NAME KERNEL_REGEX bench-args...
name=$1; kre=$2; shift 2
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out /tmp/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -c 1 -o /tmp/ncu/$name -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --gen-workers 1 "$@" > gpurun_out/ncu_$name.log 2>&1; echo "ncu $name rc=$?"
ncu -i /tmp/ncu/$name.ncu-rep --page details --csv > gpurun_out/ncu_${name}_details.csv 2>&1
ncu -i /tmp/ncu/$name.ncu-rep --page raw --csv > gpurun_out/ncu_${name}_raw.csv 2>&1
ncu -i /tmp/ncu/$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_${name}_src.csv 2>&1
python profiles/srcagg.py gpurun_out/ncu_${name}_src.csv 40 > gpurun_out/ncu_${name}_srcagg.txt 2>&1
gzip -f gpurun_out/ncu_${name}_src.csv
ls -la gpurun_out | grep ncu_$name

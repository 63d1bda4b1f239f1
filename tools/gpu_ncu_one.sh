# usage: bash tools/gpu_ncu_one.sh <name> <config> <kernel-regex> [skip]
set -x
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$3" -s ${4:-0} -c 1 \
  -o gpurun_out/ncu/$1 -f python tools/prof_run.py $2 1 > gpurun_out/ncu/$1.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu/$1.ncu-rep --page raw --csv > gpurun_out/ncu/$1.raw.csv 2>/dev/null
ncu -i gpurun_out/ncu/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/$1.source.csv 2>/dev/null
rm -f gpurun_out/ncu/$1.ncu-rep

# usage: bash tools/gpu_ncu_cmd.sh <name> <kernel-regex> <skip> <command...>
set -x
name=$1; kre=$2; skip=$3; shift 3
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s $skip -c 1 \
  -o gpurun_out/ncu/$name -f "$@" > gpurun_out/ncu/$name.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/ncu/$name.ncu-rep --page raw --csv > gpurun_out/ncu/$name.raw.csv 2>/dev/null
ncu -i gpurun_out/ncu/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/$name.source.csv 2>/dev/null
rm -f gpurun_out/ncu/$name.ncu-rep

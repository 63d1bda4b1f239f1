# round-2 measurement pass: default bench line, cfg1 batch sweep, ncu captures of the changed
# kernels, the launch list of the bench command, full-config parity
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --config cfg1 --no-extra --no-dropin --batch-sweep > gpurun_out/final/bench_cfg1_sweep.log 2>&1; echo "sweep rc=$?"
export BF_BENCH_NO_PROFILER=1
cap() {
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$3" -s ${4:-0} -c 1 \
    -o gpurun_out/final/$1 -f python tools/prof_run.py $2 1 > gpurun_out/final/$1.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i gpurun_out/final/$1.ncu-rep --page raw --csv > gpurun_out/final/$1.raw.csv 2>/dev/null
  ncu -i gpurun_out/final/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/final/$1.source.csv 2>/dev/null
  rm -f gpurun_out/final/$1.ncu-rep
}
cap cfg3_svd_rr cfg3 "svd_rr_kernel"
cap cfg3_svd_rr_v cfg3 svd_rr_vcol_kernel
cap cfg4_svd_rr_inner cfg4 "svd_rr_kernel" 3
cap cfg4d_svd_rr_vcol cfg4d svd_rr_vcol_kernel 3
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/final/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-dropin \
  > gpurun_out/final/launches_bench.log 2>&1; echo "launch list rc=$?"
unset BF_BENCH_NO_PROFILER
timeout 1500 python tools/parity_full.py --out gpurun_out/final/parity.json > gpurun_out/final/parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/final/parity.log | cut -c1-300
du -sh gpurun_out/final

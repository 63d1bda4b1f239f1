# Round-2 ncu captures: one `ncu --set full` per config's dominant kernel(s), exported to CSV,
# plus the launch list of the default bench command (per-launch durations, cold/serialised).
set -x
export BF_BENCH_NO_PROFILER=1
mkdir -p gpurun_out/ncu2
cap() {  # name config kernel-regex launch-skip
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$3" -s ${4:-0} -c 1 \
    -o gpurun_out/ncu2/$1 -f python tools/prof_run.py $2 1 > gpurun_out/ncu2/$1.log 2>&1; echo "ncu $1 rc=$?"
}
cap cfg1_svd_reg cfg1 svd_reg_kernel
cap cfg3_svd_rr cfg3 "svd_rr_kernel"
cap cfg3_svd_rr_v cfg3 svd_rr_vkernel
cap cfg2_qr_reg cfg2 qr_reg_kernel
cap cfg4_bj_gram_mma cfg4 bj_gram_mma 3
cap cfg4_svd_rr_inner cfg4 "svd_rr_kernel" 3
cap cfg4_bj_rot_mma cfg4 bj_rot_mma 3
cap cfg4d_bj_dqr_reg cfg4d bj_dqr_reg 3
cap cfg4d_bj_dapply_wy cfg4d bj_dapply_wy 3
cap cfg5_gemm_mma cfg5 gemm_mma_kernel 1
cap cfg5_svd_rr_v cfg5 svd_rr_vkernel
for f in gpurun_out/ncu2/*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $f --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > $b.source.csv 2>/dev/null
done
rm -f gpurun_out/ncu2/*.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/ncu2/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-dropin \
  > gpurun_out/ncu2/launches_bench.log 2>&1; echo "launch list rc=$?"
du -sh gpurun_out/ncu2

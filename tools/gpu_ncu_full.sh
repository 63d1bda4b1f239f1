# One `ncu --set full` capture per config's dominant kernel (single GPU, -c 1).
set -x
mkdir -p gpurun_out/ncu
cap() {  # name config kernel-regex launch-skip
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$3" -s ${4:-0} -c 1 \
    -o gpurun_out/ncu/$1 -f python tools/prof_run.py $2 1 > gpurun_out/ncu/$1.log 2>&1; echo "ncu $1 rc=$?"
}
cap cfg3_svd_reg cfg3 svd_reg_kernel
cap cfg1_svd_reg cfg1 svd_reg_kernel
cap cfg2_qr_reg cfg2 qr_reg_kernel
cap cfg4_svd_reg cfg4 svd_reg_kernel 3
cap cfg4_bj_rot cfg4 bj_rot 3
cap cfg4_bj_gram cfg4 bj_gram 3
cap cfg5_qr_reg cfg5 qr_reg_kernel
cap cfg5_svd_reg cfg5 svd_reg_kernel
cap cfg5_gemm cfg5 gemm_kernel 2
ls -la gpurun_out/ncu
# export the pages we read (the .ncu-rep files are too large to bring back all at once)
for f in gpurun_out/ncu/*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $f --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > $b.source.csv 2>/dev/null
done
du -sh gpurun_out/ncu/*
mkdir -p gpurun_out/ncu_rep_keep
mv gpurun_out/ncu/cfg3_svd_reg.ncu-rep gpurun_out/ncu_rep_keep/ 2>/dev/null
rm -f gpurun_out/ncu/*.ncu-rep
du -sh gpurun_out

# Round measurement: GPU tests, bench (full, with CPU baselines), ncu launch lists per config
# (the bench command for the headline), one ncu --set full of the headline kernel.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1; echo "ncu bench rc=$?"
for c in cfg1 cfg2 cfg3 cfg4 cfg4d cfg5; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$c.csv python tools/prof_run.py $c 2 > /dev/null 2>&1; echo "ncu $c rc=$?"
done
bash tools/gpu_ncu_one.sh cfg3_svd_rr cfg3 "svd_rr_kernel"
bash tools/gpu_ncu_one.sh cfg3_svd_rr_v cfg3 "svd_rr_vkernel"
bash tools/gpu_ncu_one.sh cfg2_qr_reg2 cfg2 "qr_reg_kernel"
bash tools/gpu_ncu_one.sh cfg4_bj_rot_mma cfg4 "bj_rot_mma" 3
bash tools/gpu_ncu_one.sh cfg5_gemm_mma cfg5 "gemm_mma" 1
bash tools/gpu_ncu_one.sh cfg4d_dqr_reg cfg4d "bj_dqr_reg" 2
bash tools/gpu_ncu_one.sh cfg4d_dapply_wy cfg4d "bj_dapply_wy" 2
PYTHONPATH=. timeout 900 python tools/h2_timing.py --ns 4096,8192,16384,32768 --reps 3 --kinds full,rsvd --oracle-max-n 16384 --out gpurun_out/h2_timing.jsonl > gpurun_out/h2_timing.log 2>&1; echo "h2 rc=$?"

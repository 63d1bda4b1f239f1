# round-2 first box call: GPU tests (timed), full-config parity, default bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
( time timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > gpurun_out/pytest_r2a.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_r2a.log
( time timeout 1500 python tools/parity_full.py --out gpurun_out/parity_r2a.json ) > gpurun_out/parity_r2a.log 2>&1; echo "parity rc=$?"; tail -30 gpurun_out/parity_r2a.log | cut -c1-400
timeout 900 python bench.py > gpurun_out/bench_r2a.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/bench_r2a.log | cut -c1-3000

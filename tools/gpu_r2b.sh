# round-2: sampler bitwise tests + accuracy diagnostics
nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
( time timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_r2b.log
timeout 900 python tools/diag_accuracy.py > gpurun_out/diag_r2b.log 2>&1; echo "diag rc=$?"; cat gpurun_out/diag_r2b.log | cut -c1-3000

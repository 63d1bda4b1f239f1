# round-2: GPU tests + full-config parity + headline bench after the rotation fix
( time timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > gpurun_out/pytest_r2h.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_r2h.log
( time timeout 1500 python tools/parity_full.py --out gpurun_out/parity_r2h.json ) > gpurun_out/parity_r2h.log 2>&1; echo "parity rc=$?"; tail -25 gpurun_out/parity_r2h.log | cut -c1-300
timeout 600 python bench.py --no-extra --no-cpu > gpurun_out/bench_r2h.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r2h.log | cut -c1-400

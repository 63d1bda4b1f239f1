# round-2 refresh: default bench line (driver command), full GPU test suite, full parity
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/final2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final2/bench.log 2>&1; echo "bench rc=$?"
( time timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider ) > gpurun_out/final2/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/final2/pytest.log
timeout 1500 python tools/parity_full.py --out gpurun_out/final2/parity.json > gpurun_out/final2/parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/final2/parity.log | cut -c1-200

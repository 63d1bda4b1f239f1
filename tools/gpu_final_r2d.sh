# last round-2 pass on the final code: default bench line, full GPU test suite, smoke
export PYTHONUNBUFFERED=1
O=gpurun_out/final5
mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; echo "bench rc=$?"
( time timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider ) > $O/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" $O/pytest.log | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log

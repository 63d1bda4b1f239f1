# quick iteration: GPU tests (subset via $K), headline bench, parity subset
( timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "${K:-not full_config}" ) > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_q.log | cut -c1-300
for c in ${BENCH:-cfg3}; do
  timeout 600 python bench.py --config $c --no-extra --no-cpu --no-dropin --steps 10 --warmup 3 > gpurun_out/bench_q_$c.log 2>&1
  python - $c <<'PY'
import json,sys
c=sys.argv[1]
l=[x for x in open(f"gpurun_out/bench_q_{c}.log") if x.startswith("{")]
if not l: print(open(f"gpurun_out/bench_q_{c}.log").read()[-1500:]); sys.exit()
d=json.loads(l[-1]); r=d["roofline"]
print(c, "value %.0f ms %.3f frac %.3f e2e %.0f" % (d["value"], d["ms_per_step"], r["frac"], d["e2e"]["value"]), d.get("kernels_per_step"))
PY
done
if [ -n "$PARITY" ]; then timeout 1200 python tools/parity_full.py --configs $PARITY --out gpurun_out/parity_q.json > gpurun_out/parity_q.log 2>&1; echo "parity rc=$?"; tail -4 gpurun_out/parity_q.log | cut -c1-400; fi

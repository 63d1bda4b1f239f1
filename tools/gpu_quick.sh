# quick check: svd parity tests + headline bench without the CPU legs
set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "svd or block or rsvd" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_q.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_q.log 2>&1; echo "bench rc=$?"
python - <<'P'
import json
l=[x for x in open('gpurun_out/bench_q.log') if x.startswith('{')][-1]
d=json.loads(l)
print("HEADLINE", d["config"]["config"], round(d["value"]), "mat/s", round(d["ms_per_step"],3), "ms", "frac", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"]))
for k,v in d.get("configs",{}).items(): print(k, round(v["value"]), "mat/s", round(v["ms_per_step"],3), "ms fp64_frac", round(v["fp64_frac"],3))
P

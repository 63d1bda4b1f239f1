# A/B timing of library variants: VARS="default name ..." CFGS="cfg3 ..." bash tools/gpu_ab.sh
for v in ${VARS:-default}; do
  if [ $v = default ]; then unset BATCHFACT_B200_LIB; else export BATCHFACT_B200_LIB=$PWD/var_libs/lib_$v.so; fi
  for c in ${CFGS:-cfg3}; do
    timeout 600 python bench.py --config $c --no-extra --no-cpu --no-dropin --steps ${STEPS:-10} --warmup 3 > gpurun_out/ab_${v}_$c.log 2>&1
    python - $v $c <<'PY'
import json,sys
v,c=sys.argv[1:3]
l=[x for x in open(f"gpurun_out/ab_{v}_{c}.log") if x.startswith("{")]
if not l: print(v, c, "FAILED", open(f"gpurun_out/ab_{v}_{c}.log").read()[-800:]); sys.exit()
d=json.loads(l[-1]); r=d["roofline"]
print(v, c, "ms %.3f frac %.3f" % (d["ms_per_step"], r["frac"]))
PY
  done
done

for v in ${VARS:-default rot}; do
  if [ $v = default ]; then unset BATCHFACT_B200_LIB; else export BATCHFACT_B200_LIB=$PWD/var_libs/lib_$v.so; fi
  echo "== $v"; timeout 300 python tools/diag_accuracy.py quick 2>&1 | python -c "
import sys, json
for ln in sys.stdin:
    try: d = json.loads(ln)
    except Exception: print(ln.strip()[:300]); continue
    for k, v in d.items():
        if k.startswith('cfg4d'): print(k, json.dumps(v)); continue
        for t, r in v.items(): print(k, t, 'orth_v p50 %.3e' % r['orth_v'][0], 'recon p50 %.3e' % r['recon'][0], 'vbias %.3e' % r['vnorm_bias'][0], 'rot %.1f sw %.2f' % (r['rotations'], r['sweeps']))
"
done

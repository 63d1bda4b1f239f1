timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
python tools/time_variants.py 2>&1 | grep "tier=auto"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('HEADLINE', round(d['value']), round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']))
for k,v in d['configs'].items(): print(k, round(v['value']), round(v['ms_per_step'],3), 'fp64', round(v['fp64_frac'],3))"

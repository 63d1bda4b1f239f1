timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "qr or rsvd or make_matrix or block" 2>&1 | tail -2
for v in loop unrolled; do
 if [ $v = unrolled ]; then export BF_QR_UNROLLED=1; fi
 echo "== $v"
 timeout 600 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu --no-extra 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', round(d['value']), d['ms_per_step'])"
 timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu --no-extra 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', round(d['value']), d['ms_per_step'])"
done

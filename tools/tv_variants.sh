timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rsvd or make_matrix or gauss or pipeline" 2>&1 | tail -2
timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu --no-extra 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', round(d['value']), d['ms_per_step'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg5_g.csv python tools/prof_run.py cfg5 1 > /dev/null 2>&1

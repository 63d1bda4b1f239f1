# round-2 measurement refresh after the float32 / TMA / drop-in changes: default bench line,
# ncu captures of the tensor-map TMA block kernels, launch list of the bench command, full GPU
# test suite, full-config parity (float64 and float32 twins), smoke
export PYTHONUNBUFFERED=1
O=gpurun_out/final3
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.log 2>&1; echo "bench rc=$?"
export BF_BENCH_NO_PROFILER=1
cap() {
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$3" -s ${4:-0} -c 1 \
    -o $O/$1 -f python tools/prof_run.py $2 1 > $O/$1.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1.raw.csv 2>/dev/null
  ncu -i $O/$1.ncu-rep --page source --csv --print-source sass > $O/$1.source.csv 2>/dev/null
  rm -f $O/$1.ncu-rep
}
cap cfg4_bj_gram_tma cfg4 bj_gram_tma 3
cap cfg4_bj_rot_tma cfg4 bj_rot_tma 3
cap cfg4d_bj_rot_tma cfg4d bj_rot_tma 3
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-dropin \
  > $O/launches_bench.log 2>&1; echo "launch list rc=$?"
unset BF_BENCH_NO_PROFILER
( time timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider ) > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 1500 python tools/parity_full.py --out $O/parity.json > $O/parity.log 2>&1; echo "parity rc=$?"; tail -1 $O/parity.log | cut -c1-200
timeout 900 python tools/parity_full.py --configs cfg1f32,cfg1rrf32,cfg2f32,cfg3f32,cfg4df32,cfg5f32 --out $O/parity_f32.json > $O/parity_f32.log 2>&1; echo "parity f32 rc=$?"; tail -1 $O/parity_f32.log | cut -c1-200
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
du -sh $O

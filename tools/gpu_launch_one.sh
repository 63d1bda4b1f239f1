# launch list of one hot-path call per config: CFGS="cfg5 cfg4d" bash tools/gpu_launch_one.sh
export BF_BENCH_NO_PROFILER=1
for c in ${CFGS:-cfg5}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_$c.csv python tools/prof_run.py $c 2 > /dev/null 2>&1; echo "$c rc=$?"
  python tools/launch_summary.py gpurun_out/launches_$c.csv | head -14
done

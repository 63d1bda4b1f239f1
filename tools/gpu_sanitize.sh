set -x
for tool in racecheck memcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc=$?"
  tail -3 gpurun_out/sanitize_$tool.log
done
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "svd or rsvd" 2>&1 | tail -1

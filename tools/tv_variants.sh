./tools/microbench/rot_latency
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "svd or rsvd or block" 2>&1 | tail -3
python tools/time_variants.py 2>&1 | grep "tier=auto"

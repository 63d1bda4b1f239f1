timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "svd or block or rsvd" 2>&1 | tail -5
python tools/time_variants.py 2>&1 | grep "tier=auto" | grep -v serial

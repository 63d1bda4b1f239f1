timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "block" 2>&1 | tail -3
python tools/time_block.py

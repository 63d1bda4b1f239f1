python tools/time_block.py
python tools/time_block.py

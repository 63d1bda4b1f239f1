( time timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_config" ) > gpurun_out/pytest_r2i.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_r2i.log | cut -c1-400
( time timeout 1500 python tools/parity_full.py --out gpurun_out/parity_r2i.json ) > gpurun_out/parity_r2i.log 2>&1; echo "parity rc=$?"; tail -12 gpurun_out/parity_r2i.log | cut -c1-300

timeout 600 python -m pytest tests/test_gpu_slabs.py -x -q -m gpu -k "error or two_processes" 2>&1 | tail -3
bash scripts/r2_prof.sh base wet
python scripts/quick_perf.py wet 2048 40 1 2>&1 | tail -1

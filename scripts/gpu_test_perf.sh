set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
python scripts/quick_perf.py c2 2048 40 1
python scripts/quick_perf.py wet 2048 40 1
python scripts/quick_perf.py c1 256 200 1

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
python -c "import torch; print(torch.cuda.is_available())"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -30
python scripts/quick_perf.py c2 2048 40 1
python scripts/quick_perf.py c2 2048 40 0
python scripts/quick_perf.py wet 2048 40 1
python scripts/quick_perf.py c1 256 200 1

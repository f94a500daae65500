# parity tests (fast subset first) + quick device timing of c2 and the fully wet grid
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_${TAG}.log
python scripts/quick_perf.py c2 2048 40 1 2>&1 | tail -1
python scripts/quick_perf.py wet 2048 40 1 2>&1 | tail -1

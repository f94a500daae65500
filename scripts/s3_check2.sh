TAG=${1:-x}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_${TAG}.log
for i in 1 2; do timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k c4_peer 2>&1 | tail -1; done
for gs in 16 64; do
  python scripts/quick_perf.py c3 4096 400 1 $gs 2>&1 | tail -1
  python scripts/quick_perf.py c1 256 1000 1 $gs 2>&1 | tail -1
  python scripts/quick_perf.py c2 2048 200 1 $gs 2>&1 | tail -1
done

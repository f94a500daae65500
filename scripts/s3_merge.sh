TAG=${1:-x}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; tail -2 gpurun_out/pytest_${TAG}.log
for r in 1 2; do
for o in "merge_post=0" "merge_post=1"; do
  echo "$o $(QP_OPTS=$o python scripts/quick_perf.py c3 4096 400 1 16 2>&1 | tail -1)"
  echo "$o $(QP_OPTS=$o python scripts/quick_perf.py c1 256 1000 1 16 2>&1 | tail -1)"
  echo "$o $(QP_OPTS=$o python scripts/quick_perf.py c2 2048 200 1 16 2>&1 | tail -1)"
done; done | tee gpurun_out/merge_${TAG}.txt

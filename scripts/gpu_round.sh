# tests + quick perf + ncu capture of the stage kernels (one gpurun call)
TAG=${1:-x}
set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -12
python scripts/quick_perf.py c2 2048 40 1
python scripts/quick_perf.py wet 2048 40 1
mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 8 -c 2 \
    -o gpurun_out/prof_${TAG} python scripts/quick_perf.py c2 2048 4 1 4 > gpurun_out/prof_${TAG}.log 2>&1

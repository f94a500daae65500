# ncu capture of the stage kernels (run under gpurun; one GPU).
set -x
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
TAG=${1:-r1}
SC=${2:-c2}
N=${3:-2048}
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python scripts/quick_perf.py $SC $N 4 1 4 > gpurun_out/launches_${TAG}.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:stage_kernel -s 8 -c 2 \
    -o gpurun_out/prof_${TAG} python scripts/quick_perf.py $SC $N 4 1 4 > gpurun_out/prof_${TAG}.log 2>&1
ls -la gpurun_out

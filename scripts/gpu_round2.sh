TAG=${1:-x}
set -x
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -12
python -c "import __graft_entry__ as g; g.smoke()"
mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
   python bench.py --steps 8 --warmup 3 --no-cpu --roofline-reps 1 > gpurun_out/launches_${TAG}.log 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 30 -c 2 \
    -o gpurun_out/prof_${TAG} python bench.py --steps 8 --warmup 3 --no-cpu --roofline-reps 1 > gpurun_out/prof_${TAG}.log 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 30 -c 2 \
    -o gpurun_out/prof_${TAG}_wet python bench.py --config wet --steps 8 --warmup 3 --no-cpu --roofline-reps 1 > gpurun_out/prof_${TAG}_wet.log 2>&1

TAG=${1:-x}
mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 30 -c 2 \
    -o gpurun_out/prof_${TAG}_wet python bench.py --config wet --steps 8 --warmup 3 --no-cpu --roofline-reps 1 > gpurun_out/prof_${TAG}_wet.log 2>&1

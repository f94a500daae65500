# ncu --set full of the two stage kernels on one config (default wet) + quick timings
TAG=${1:-x}; CFG=${2:-wet}; N=${3:-2048}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:stage_kernel -s 30 -c 2 \
    -o gpurun_out/prof_${TAG}_${CFG} python bench.py --config $CFG --ncols $N --nrows $N --steps 8 --warmup 3 --no-cpu --no-extra --roofline-reps 1 > gpurun_out/prof_${TAG}_${CFG}.log 2>&1
echo ncu_rc=$?

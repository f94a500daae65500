# C3 (sparse, Mode-II) timing + ncu --set full of its wide stage kernels + the A/B of variants
TAG=${1:-x}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python bench.py --config c3 --ncols 4096 --nrows 2048 --steps 400 --warmup 10 --no-cpu --no-extra > gpurun_out/c3_${TAG}.json 2> gpurun_out/c3_${TAG}.err
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:stage_kernel -s 60 -c 2 \
    -o gpurun_out/prof_${TAG}_c3 python bench.py --config c3 --ncols 4096 --nrows 2048 --steps 40 --warmup 3 --no-cpu --no-extra --roofline-reps 1 > gpurun_out/prof_${TAG}_c3.log 2>&1
echo ncu_rc=$?
[ -n "$VARIANTS" ] && bash scripts/gpu_abn.sh ${2:-200} ${3:-2}

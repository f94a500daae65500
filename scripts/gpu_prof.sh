# ncu --set full of the two stage kernels (c2 and fully wet) with source + the launch list, one GPU
TAG=${1:-x}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for cfg in c2 wet; do
$NCU --set full --clock-control none --import-source on -k regex:stage_kernel -s 30 -c 2 \
    -o gpurun_out/prof_${TAG}_${cfg} python bench.py --config $cfg --steps 8 --warmup 3 --no-cpu --no-extra --roofline-reps 1 > gpurun_out/prof_${TAG}_${cfg}.log 2>&1
done
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
   python bench.py --steps 8 --warmup 3 --no-cpu --no-extra --roofline-reps 1 > gpurun_out/launches_${TAG}.log 2>&1
ls -la gpurun_out | tail -6

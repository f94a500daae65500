# session-3 profiling: FP64 probe, ncu --set full (source) of the wet stage kernels, C3 launch list
TAG=${1:-x}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
./scripts/probes/bin/fp64_probe > gpurun_out/fp64_${TAG}.txt 2>&1
python scripts/quick_perf.py c3 4096 400 1 > gpurun_out/qp_c3_${TAG}.txt 2>&1
python scripts/quick_perf.py wet 2048 200 1 >> gpurun_out/qp_c3_${TAG}.txt 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_${TAG}.csv \
   python bench.py --config c3 --ncols 4096 --nrows 2048 --steps 30 --warmup 3 --no-cpu --no-extra --roofline-reps 1 > gpurun_out/launches_c3_${TAG}.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:stage_kernel -s 30 -c 2 \
    -o gpurun_out/prof_${TAG}_wet python bench.py --config wet --steps 8 --warmup 3 --no-cpu --no-extra --roofline-reps 1 > gpurun_out/prof_${TAG}_wet.log 2>&1
echo ncu_rc=$?

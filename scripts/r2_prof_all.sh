# round-2 profiles: ncu --set full of the stage kernels on c2, wet (2048^2) and c5 (8192^2) + launch list
TAG=${1:-r2}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for spec in c2:c2:2048 wet:wet:2048 c5:c2:8192; do
  name=${spec%%:*}; rest=${spec#*:}; cfg=${rest%%:*}; n=${rest#*:}
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:stage_kernel -s 30 -c 2 \
    -o gpurun_out/prof_${TAG}_${name} python bench.py --config $cfg --ncols $n --nrows $n --steps 8 --warmup 3 --no-cpu --no-extra --roofline-reps 1 > gpurun_out/prof_${TAG}_${name}.log 2>&1
  echo "$name ncu rc=$?"
done
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
   python bench.py --steps 8 --warmup 3 --no-cpu --no-extra --roofline-reps 1 > gpurun_out/launches_${TAG}.log 2>&1
echo "launches rc=$?"

# our arm and the reference arm per config (one GPU)
mkdir -p gpurun_out
for spec in c1:256:256 c2:2048:2048 c3:4096:2048 c4:6000:4000 c2:8192:8192; do
  cfg=${spec%%:*}; rest=${spec#*:}; nc=${rest%%:*}; nr=${rest#*:}
  steps=200; [ $nc -ge 6000 ] && steps=40
  python bench.py --config $cfg --ncols $nc --nrows $nr --steps $steps --warmup 5 --no-extra --cpu-steps 6 > gpurun_out/tab_${cfg}_${nc}.json 2> gpurun_out/tab_${cfg}_${nc}.err
  echo "$cfg $nc x $nr rc=$?"
  python bench.py --impl reference --config $cfg --ncols $nc --nrows $nr --steps 6 --warmup 3 --no-extra > gpurun_out/tabref_${cfg}_${nc}.json 2> gpurun_out/tabref_${cfg}_${nc}.err
  echo "ref rc=$?"
done

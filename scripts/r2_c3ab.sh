# C3 sparse-step timing, base vs current library
for v in ${VARIANTS:-base cur}; do
  if [ "$v" = cur ]; then L=$PWD/paper_2104_06784_b200/libtpflow_b200.so; else L=$PWD/paper_2104_06784_b200/libtpflow_b200_$v.so; fi
  TPFLOW_B200_LIB=$L python bench.py --config c3 --ncols 4096 --nrows 2048 --steps 400 --warmup 10 --no-cpu --no-extra 2>&1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v c3 ms/step', d['ms_per_step'], 'GCUPS', d['value'], 'tiles', d['config']['active_tiles_last_step'], 'launches', d['gpu_launches'])"
done

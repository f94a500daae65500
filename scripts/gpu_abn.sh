# A/B/n device timing of library variants on the same box (development aid):
#   VARIANTS="base cap2 cap3" CFGS="c2 wet" bash scripts/gpu_abn.sh [steps] [reps]
# variant "cur" is the built library; others are paper_2104_06784_b200/libtpflow_b200_<name>.so
STEPS=${1:-100}
REPS=${2:-2}
for r in $(seq $REPS); do
  for cfg in ${CFGS:-c2 wet}; do
    for v in ${VARIANTS:-base cur}; do
      if [ "$v" = cur ]; then L=$PWD/paper_2104_06784_b200/libtpflow_b200.so; else L=$PWD/paper_2104_06784_b200/libtpflow_b200_$v.so; fi
      echo "$v $(TPFLOW_B200_LIB=$L python scripts/quick_perf.py $cfg 2048 $STEPS 1 2>&1 | tail -1)"
    done
  done
done

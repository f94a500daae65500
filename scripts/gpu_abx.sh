# A/B device timing: paper_2104_06784_b200/libtpflow_b200_base.so (A) vs the built library (B),
# alternating on the same box; usage: bash scripts/gpu_abx.sh [steps] [reps]
STEPS=${1:-100}
REPS=${2:-3}
A=paper_2104_06784_b200/libtpflow_b200_base.so
B=paper_2104_06784_b200/libtpflow_b200.so
for r in $(seq $REPS); do
  for cfg in ${CFGS:-c2 wet}; do
    echo "A $(TPFLOW_B200_LIB=$PWD/$A python scripts/quick_perf.py $cfg 2048 $STEPS 1 2>&1 | tail -1)"
    echo "B $(TPFLOW_B200_LIB=$PWD/$B python scripts/quick_perf.py $cfg 2048 $STEPS 1 2>&1 | tail -1)"
  done
done

# C3 + C2 A/B/n of library variants: VARIANTS="cur x" bash scripts/s3_c3ab.sh TAG [steps] [reps]
TAG=${1:-x}
mkdir -p gpurun_out
for r in $(seq ${3:-2}); do
  for v in ${VARIANTS:-cur}; do
    if [ "$v" = cur ]; then L=$PWD/paper_2104_06784_b200/libtpflow_b200.so; else L=$PWD/paper_2104_06784_b200/libtpflow_b200_$v.so; fi
    echo "$v $(TPFLOW_B200_LIB=$L python scripts/quick_perf.py c3 4096 ${2:-400} 1 2>&1 | tail -1)"
    echo "$v $(TPFLOW_B200_LIB=$L python scripts/quick_perf.py c2 2048 200 1 2>&1 | tail -1)"
  done
done | tee gpurun_out/c3ab_${TAG}.txt

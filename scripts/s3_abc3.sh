# A/B/n of variants on C3, C1, C2: VARIANTS="base cur x" bash scripts/s3_abc3.sh TAG [reps]
TAG=${1:-x}
mkdir -p gpurun_out
for r in $(seq ${2:-2}); do
  for v in ${VARIANTS:-base cur}; do
    if [ "$v" = cur ]; then L=$PWD/paper_2104_06784_b200/libtpflow_b200.so; else L=$PWD/paper_2104_06784_b200/libtpflow_b200_$v.so; fi
    echo "$v $(TPFLOW_B200_LIB=$L python scripts/quick_perf.py c3 4096 400 1 16 2>&1 | tail -1)"
    echo "$v $(TPFLOW_B200_LIB=$L python scripts/quick_perf.py c1 256 1000 1 16 2>&1 | tail -1)"
    echo "$v $(TPFLOW_B200_LIB=$L python scripts/quick_perf.py c2 2048 200 1 16 2>&1 | tail -1)"
  done
done | tee gpurun_out/abc3_${TAG}.txt

# parity of a variant library (GPU tests with TPFLOW_B200_LIB) then A/B/n timing
# usage: VAR=dual VARIANTS="cur dual" CFGS="c2 wet" bash scripts/s3_abn.sh TAG [steps] [reps]
TAG=${1:-x}
mkdir -p gpurun_out
if [ -n "$VAR" ]; then
  TPFLOW_B200_LIB=$PWD/paper_2104_06784_b200/libtpflow_b200_$VAR.so timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_${TAG}.log
fi
bash scripts/gpu_abn.sh ${2:-200} ${3:-3} > gpurun_out/ab_${TAG}.txt 2>&1; cat gpurun_out/ab_${TAG}.txt

# parity (GPU tests) then A/B timing of libtpflow_b200_base.so vs the built library
TAG=${1:-x}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_${TAG}.log
CFGS="${CFGS:-c2 wet}" bash scripts/gpu_abx.sh ${STEPS:-200} ${REPS:-3} > gpurun_out/ab_${TAG}.txt 2>&1; cat gpurun_out/ab_${TAG}.txt

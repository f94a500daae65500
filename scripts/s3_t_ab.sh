# GPU tests, then A/B/n (C3, C1, C2) + wet of library variants
TAG=${1:-x}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_${TAG}.log
bash scripts/s3_abc3.sh ${TAG} ${REPS:-2}
CFGS=wet bash scripts/gpu_abn.sh 100 2

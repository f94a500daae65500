# parity subset + A/B timing (base .so vs built)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
bash scripts/gpu_abx.sh ${1:-100} ${2:-2}

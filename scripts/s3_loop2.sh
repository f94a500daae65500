for o in "device_loop=0" "device_loop=2" "device_loop=1"; do
  echo "$o $(QP_OPTS=$o python scripts/quick_perf.py c1 256 1000 1 16 2>&1 | tail -1)"
  echo "$o $(QP_OPTS="$o wide_tiles=0" python scripts/quick_perf.py c1 256 1000 1 16 2>&1 | tail -1)"
  echo "$o $(QP_OPTS=$o python scripts/quick_perf.py c3 4096 400 1 8 2>&1 | tail -1)"
done
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k c4_peer 2>&1 | tail -1; done

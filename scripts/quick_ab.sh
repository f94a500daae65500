set -x
for k in 2 3; do
  TP_KERNEL=$k python scripts/quick_perf.py c2 2048 40 1
  TP_KERNEL=$k python scripts/quick_perf.py wet 2048 40 1
done

for gs in 1 2 4 8 16 32; do python scripts/quick_perf.py c3 4096 400 1 $gs 2>&1 | tail -1; done
for gs in 4 16; do python scripts/quick_perf.py c2 2048 200 1 $gs 2>&1 | tail -1; done

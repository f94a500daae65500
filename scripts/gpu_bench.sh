set -x
python bench.py 2>&1 | tail -3
python bench.py --impl reference --steps 20 2>&1 | tail -2

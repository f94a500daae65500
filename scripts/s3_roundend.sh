# what the driver runs at round end: GPU tests (twice, flakiness), smoke(), default bench (both arms)
TAG=${1:-x}
mkdir -p gpurun_out
for i in 1 2; do timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${TAG}_$i.log 2>&1; tail -1 gpurun_out/pytest_${TAG}_$i.log; done
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -c 300 gpurun_out/bench_${TAG}.json
timeout 900 python bench.py --impl reference > gpurun_out/ref_${TAG}.json 2> gpurun_out/ref_${TAG}.err; tail -c 200 gpurun_out/ref_${TAG}.json

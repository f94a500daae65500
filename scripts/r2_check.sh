# round-2 check: GPU tests, default bench (both arms), a functional 2-rank strong-scaling run
TAG=${1:-x}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; tail -5 gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -c 3000 gpurun_out/bench_${TAG}.json; tail -5 gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_${TAG}.json 2> gpurun_out/ref_${TAG}.err; cat gpurun_out/ref_${TAG}.json; tail -5 gpurun_out/ref_${TAG}.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 6 --warmup 3 --scaling strong --config c4 --ncols 600 --nrows 400 --no-cpu > gpurun_out/n2s_${TAG}.json 2> gpurun_out/n2s_${TAG}.err; cat gpurun_out/n2s_${TAG}.json; tail -5 gpurun_out/n2s_${TAG}.err

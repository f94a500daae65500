# measurement refresh: ncu profiles (c2, wet, c5 + launch list), default bench (both arms), C3 line
TAG=${1:-r2b}
mkdir -p gpurun_out
bash scripts/r2_prof_all.sh $TAG
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -c 400 gpurun_out/bench_${TAG}.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_${TAG}.json 2> gpurun_out/ref_${TAG}.err; tail -c 300 gpurun_out/ref_${TAG}.json
timeout 600 python bench.py --config c3 --ncols 4096 --nrows 2048 --steps 400 --warmup 10 --no-cpu --no-extra > gpurun_out/c3_${TAG}.json 2> gpurun_out/c3_${TAG}.err
timeout 600 python bench.py --config c4 --ncols 6000 --nrows 4000 --steps 100 --warmup 10 --no-cpu --no-extra > gpurun_out/c4_${TAG}.json 2> gpurun_out/c4_${TAG}.err
timeout 600 python bench.py --config wet --steps 50 --warmup 5 --no-cpu --no-extra > gpurun_out/wet_${TAG}.json 2> gpurun_out/wet_${TAG}.err
ls gpurun_out | grep $TAG

mkdir -p gpurun_out
(free -g; nproc; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv) > gpurun_out/r2_box.txt 2>&1
./scripts/probes/fp64_probe > gpurun_out/r2_fp64_probe.txt 2>&1
python scripts/quick_perf.py wet 2048 40 1 > gpurun_out/r2_qp_base.txt 2>&1
python scripts/quick_perf.py c2 2048 40 1 >> gpurun_out/r2_qp_base.txt 2>&1
cat gpurun_out/r2_box.txt gpurun_out/r2_fp64_probe.txt gpurun_out/r2_qp_base.txt

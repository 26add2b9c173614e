set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
./tools/l2_bench > gpurun_out/r2a_l2_bench.json 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench_c4.json 2> gpurun_out/r2a_bench_c4.err
tail -3 gpurun_out/r2a_bench_c4.err
cat gpurun_out/r2a_bench_c4.json

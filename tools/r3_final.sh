# final check of the build: default bench, launch list of the bench's sweep kernels, smoke, full GPU suite
export PYTHONDONTWRITEBYTECODE=1
export MFG_SYNTH_CACHE=/tmp/synth
tag=${TAG:-r3g}
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -c 400 gpurun_out/${tag}_bench.json; tail -2 gpurun_out/${tag}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_bench_reference.json 2>&1; tail -c 600 gpurun_out/${tag}_bench_reference.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none \
    -k regex:"k_panel|k_cold|k_sweep|k_gather4|k_dot" -c 80 --csv --log-file gpurun_out/${tag}_c4_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-tto --no-bcd > gpurun_out/${tag}_launch_ncu.log 2>&1
echo "launch list rc=$?"
python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
tail -4 gpurun_out/${tag}_pytest_gpu.log

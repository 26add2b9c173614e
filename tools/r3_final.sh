# final profiles of the hybrid sweep at c4: ncu --set full of k_panel4 and k_cold4,
# launch list of the bench's sweep kernels, default bench, full GPU suite
export PYTHONDONTWRITEBYTECODE=1
export MFG_SYNTH_CACHE=/tmp/synth
tag=${TAG:-r3b}
MFG_PROBE_QUICK=1 python tools/panel_probe.py c4 > gpurun_out/${tag}_plain.log 2>&1 || { tail gpurun_out/${tag}_plain.log; exit 1; }
MFG_PROBE_QUICK=1 ncu --set full --clock-control none --import-source on -k regex:"^k_panel4$" -s 0 -c 1 -f \
    -o gpurun_out/${tag}_k_panel4 python tools/panel_probe.py c4 > gpurun_out/${tag}_ncu1.log 2>&1
echo "k_panel4 rc=$?"
MFG_PROBE_QUICK=1 ncu --set full --clock-control none --import-source on -k regex:"^k_cold4$" -s 0 -c 1 -f \
    -o gpurun_out/${tag}_k_cold4 python tools/panel_probe.py c4 > gpurun_out/${tag}_ncu2.log 2>&1
echo "k_cold4 rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -c 600 gpurun_out/${tag}_bench.json; tail -2 gpurun_out/${tag}_bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none \
    -k regex:"k_panel|k_cold|k_sweep|k_gather4|k_dot" -c 80 --csv --log-file gpurun_out/${tag}_c4_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-tto --no-bcd > gpurun_out/${tag}_launch_ncu.log 2>&1
echo "launch list rc=$?"
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
tail -4 gpurun_out/${tag}_pytest_gpu.log

# round-2 final: lmin A/B, default bench, launch list of the bench's sweep kernels, full GPU suite
export PYTHONDONTWRITEBYTECODE=1
export MFG_SYNTH_CACHE=/tmp/synth
tag=${TAG:-r2w}
for lmin in 24 32; do
  echo "== LMIN=$lmin"
  MFG_PANEL_LMIN=$lmin timeout 300 python tools/panel_probe.py c4 2>&1 | tail -2
done > gpurun_out/${tag}_lmin.log 2>&1
cat gpurun_out/${tag}_lmin.log | cut -c1-220
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -c 1500 gpurun_out/${tag}_bench.json; tail -2 gpurun_out/${tag}_bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none \
    -k regex:"k_panel|k_sweep|k_gather4" -c 60 --csv --log-file gpurun_out/${tag}_c4_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-tto --no-bcd > gpurun_out/${tag}_launch_ncu.log 2>&1
echo "launch list rc=$?"
if [ -z "$NOTESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
tail -4 gpurun_out/${tag}_pytest_gpu.log
fi

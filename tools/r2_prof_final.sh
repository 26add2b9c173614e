# round-2 profiles: launch list of the default bench (c4), ncu --set full of
# the BCD DMMA kernel (c4, CSR and CSC half-sweeps) and of the sweep at c4.
export PYTHONDONTWRITEBYTECODE=1
export MFG_SYNTH_CACHE=/tmp/synth
tag=${TAG:-r2k}
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-tto --no-bcd > gpurun_out/${tag}_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_c4_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-tto --no-bcd \
    > gpurun_out/${tag}_launch_ncu.log 2>&1
echo "launch list rc=$?"
python tools/bcd_one.py c4 40 csr > gpurun_out/${tag}_bcd_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bcd_dm -s 1 -c 1 \
    -o gpurun_out/${tag}_bcd_c4_csr python tools/bcd_one.py c4 40 csr > gpurun_out/${tag}_bcd_ncu1.log 2>&1
echo "bcd csr rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_bcd_dm -s 1 -c 1 \
    -o gpurun_out/${tag}_bcd_c4_csc python tools/bcd_one.py c4 40 csc > gpurun_out/${tag}_bcd_ncu2.log 2>&1
echo "bcd csc rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_sweep_g8f -s 3 -c 1 \
    -o gpurun_out/${tag}_sweep_c4 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-tto --no-bcd > gpurun_out/${tag}_sweep_ncu.log 2>&1
echo "sweep rc=$?"

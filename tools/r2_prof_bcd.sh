# ncu of the DMMA BCD kernel on the c4 CSC half-sweep (k=40)
export PYTHONDONTWRITEBYTECODE=1
python tools/bcd_one.py c4 40 csc > gpurun_out/r2d_bcd_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bcd_dm -s 1 -c 1 \
    -o gpurun_out/r2d_bcd_c4_csc python tools/bcd_one.py c4 40 csc > gpurun_out/r2d_bcd_ncu.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/r2d_bcd_ncu.log

# ncu --set full of the panel kernel (and its fold) at c4 through tools/panel_probe.py
export PYTHONDONTWRITEBYTECODE=1
export MFG_SYNTH_CACHE=/tmp/synth
tag=${TAG:-r2p}
MFG_PROBE_QUICK=1 python tools/panel_probe.py ${WL:-c4} > gpurun_out/${tag}_plain.log 2>&1 || { tail gpurun_out/${tag}_plain.log; exit 1; }
MFG_PROBE_QUICK=1 ncu --set full --clock-control none --import-source on -k regex:"^k_panel4?$" -s 0 -c 1 -f \
    -o gpurun_out/${tag}_k_panel python tools/panel_probe.py ${WL:-c4} > gpurun_out/${tag}_ncu.log 2>&1
echo "k_panel rc=$?"
if [ -n "$FOLD" ]; then
MFG_PROBE_QUICK=1 ncu --set full --clock-control none --import-source on -k k_panel_fold -s 0 -c 2 -f \
    -o gpurun_out/${tag}_k_panel_fold python tools/panel_probe.py ${WL:-c4} > gpurun_out/${tag}_ncu2.log 2>&1
echo "fold rc=$?"
fi
ls -la gpurun_out/${tag}_*

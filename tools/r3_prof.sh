# ncu --set full of k_panel4 and k_cold4 at c4 (final build)
export PYTHONDONTWRITEBYTECODE=1
export MFG_SYNTH_CACHE=/tmp/synth
tag=${TAG:-r3i}
MFG_PROBE_QUICK=1 python tools/panel_probe.py c4 > gpurun_out/${tag}_plain.log 2>&1 || { tail gpurun_out/${tag}_plain.log; exit 1; }
MFG_PROBE_QUICK=1 ncu --set full --clock-control none --import-source on -k regex:"^k_panel4$" -s 0 -c 1 -f \
    -o gpurun_out/${tag}_k_panel4 python tools/panel_probe.py c4 > gpurun_out/${tag}_ncu1.log 2>&1
echo "k_panel4 rc=$?"
MFG_PROBE_QUICK=1 ncu --set full --clock-control none --import-source on -k regex:"^k_cold4$" -s 0 -c 1 -f \
    -o gpurun_out/${tag}_k_cold4 python tools/panel_probe.py c4 > gpurun_out/${tag}_ncu2.log 2>&1
echo "k_cold4 rc=$?"

# parameter sweep of the hybrid plan at c4 + ncu of k_panel
export PYTHONDONTWRITEBYTECODE=1
export MFG_SYNTH_CACHE=/tmp/synth
tag=${TAG:-r2r}
for cfg in "64 100000 8 256" "128 50000 8 256" "128 50000 4 256" "64 100000 8 128" "64 100000 8 511"; do
  set -- $cfg
  echo "== MAXP=$1 MINE=$2 LMIN=$3 LMAX=$4"
  MFG_PANEL_MAXP=$1 MFG_PANEL_MINE=$2 MFG_PANEL_LMIN=$3 MFG_PANEL_LMAX=$4 timeout 300 python tools/panel_probe.py c4 2>&1 | tail -2
done > gpurun_out/${tag}_sweep.log 2>&1
cat gpurun_out/${tag}_sweep.log
MFG_PROBE_QUICK=1 ncu --set full --clock-control none --import-source on -k k_panel -s 0 -c 1 -f \
    -o gpurun_out/${tag}_k_panel python tools/panel_probe.py c4 > gpurun_out/${tag}_ncu.log 2>&1
echo "k_panel rc=$?"

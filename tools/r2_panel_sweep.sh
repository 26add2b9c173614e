# parameter sweep of the hybrid plan at c4
export PYTHONDONTWRITEBYTECODE=1
export MFG_SYNTH_CACHE=/tmp/synth
tag=${TAG:-r2r}
IFS=";" read -ra CF <<< "${CFGS:-64 100000 8 256;64 100000 12 256;32 100000 16 256;48 100000 16 256;48 100000 24 256;64 100000 16 511}"
for cfg in "${CF[@]}"; do
  set -- $cfg
  echo "== MAXP=$1 MINE=$2 LMIN=$3 LMAX=$4"
  MFG_PANEL_MAXP=$1 MFG_PANEL_MINE=$2 MFG_PANEL_LMIN=$3 MFG_PANEL_LMAX=$4 timeout 300 python tools/panel_probe.py c4 2>&1 | tail -2
done > gpurun_out/${tag}_sweep.log 2>&1
cat gpurun_out/${tag}_sweep.log

# A/B of the BCD half-sweep across the library variants in libvariants/
export MFG_SYNTH_CACHE=/tmp/mfg_synth
for args in ${BCD_AB_CASES:-"c2 20" "c2 40" "c2 100" "c2 199" "c3 30" "c3 480" "c4 40"}; do
  for l in libvariants/*.so; do
    echo "== $(basename $l) $args"; MFG_LIB_PATH=$PWD/$l timeout 600 python tools/bcd_probe.py $args 2>&1 | grep -v Warn
  done
done

#!/bin/bash
# A/B the library variants in libvariants/ on the given workloads:
#   tools/ab_libs.sh "c2 c4" [reps]
# prints kernel us (CUDA-event average of the main sweep launch) and step us.
wls=${1:-c2}
reps=${2:-2}
export MFG_SYNTH_CACHE=/tmp/mfg_synth
for wl in $wls; do
  for rep in $(seq $reps); do
    for lib in libvariants/*.so; do
      r=$(MFG_LIB_PATH=$PWD/$lib python bench.py --workload $wl --steps 100 --warmup 5 --no-cpu-baseline --no-tto 2>/dev/null \
          | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['avg_launch_us'],1), round(d['ms_per_step']*1e3,1))")
      echo "$wl rep$rep $(basename $lib .so): kernel_us step_us = $r"
    done
  done
done

#!/bin/bash
# A/B an environment knob of the current build:
#   tools/ab_env.sh VAR "v1 v2 ..." "c2 c4" [reps]
var=$1; vals=$2; wls=${3:-c2}; reps=${4:-2}
export MFG_SYNTH_CACHE=/tmp/mfg_synth
for wl in $wls; do
  for rep in $(seq $reps); do
    for v in $vals; do
      r=$(env $var=$v python bench.py --workload $wl --steps 100 --warmup 5 --no-cpu-baseline --no-tto 2>/dev/null \
          | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['avg_launch_us'],1), round(d['ms_per_step']*1e3,1), round(d['e2e']['value'],1))")
      echo "$wl rep$rep $var=$v: kernel_us step_us e2e = $r"
    done
  done
done

#!/bin/bash
for wps in 24 32 40; do
  r=$(MFG_WORKERS_PER_SM=$wps python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['avg_launch_us'],1), round(d['ms_per_step']*1e3,1))")
  echo "wps=$wps kernel_us/step_us: $r"
done

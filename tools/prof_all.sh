#!/bin/bash
# Round profiles: bench lines and one ncu --set full capture of the sweep per workload.
set -e
export MFG_SYNTH_CACHE=/tmp/mfg_synth
tag=${1:-r1d}
for wl in c2 c4 c5; do
  python bench.py --workload $wl --steps 20 --warmup 5 --no-tto --no-cpu-baseline > gpurun_out/bench_${tag}_${wl}.json 2> gpurun_out/bench_${tag}_${wl}.err
  ncu --set full --clock-control none --import-source on -k regex:k_sweep_g8f -s 8 -c 1 -f \
      -o gpurun_out/prof_${tag}_${wl} python bench.py --workload $wl --steps 3 --warmup 3 --no-tto --no-cpu-baseline \
      > gpurun_out/ncu_${tag}_${wl}.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${tag}_c2.csv \
    python bench.py --steps 3 --warmup 3 --no-tto --no-cpu-baseline > /dev/null 2>&1
echo done

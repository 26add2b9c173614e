# A/B of the sweep kernels (k_sweep_i8 vs the round-1 k_sweep_g8f, MFG_NO_I8=1)
# at c2..c5: bench.py kernel time + value, no CPU/TTO/BCD legs. Instances are
# cached under /tmp/synth within this call.
export MFG_SYNTH_CACHE=/tmp/synth
tag=${TAG:-r2b}
for wl in ${WLS:-c2 c3 c4 c5}; do
  for v in i8 g8f; do
    if [ $v = g8f ]; then export MFG_NO_I8=1; else unset MFG_NO_I8; fi
    timeout 900 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline --no-tto --no-bcd \
      > gpurun_out/${tag}_${wl}_${v}.json 2> gpurun_out/${tag}_${wl}_${v}.err
    python - "$wl" "$v" gpurun_out/${tag}_${wl}_${v}.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], "kernel_us=%.1f" % d["roofline"]["avg_launch_us"], "value=%.1f" % d["value"], "e2e=%.1f" % d["e2e"]["value"], "frac=%.3f" % d["roofline"]["frac"], d["clocks"])
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e)
PY
  done
done

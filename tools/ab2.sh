export MFG_SYNTH_CACHE=/tmp/mfg_synth
for wl in c2 c4; do for lib in libvariants/*.so; do for wps in 32 40; do
r=$(MFG_WORKERS_PER_SM=$wps MFG_LIB_PATH=$PWD/$lib python bench.py --workload $wl --steps 100 --warmup 5 --no-cpu-baseline --no-tto 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['avg_launch_us'],1))")
echo "$wl $(basename $lib) wps=$wps kernel_us=$r"
done; done; done

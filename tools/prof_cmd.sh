set -e
export MFG_SYNTH_CACHE=/tmp/mfg_synth
python bench.py --workload c2 --steps 5 --warmup 3 --no-tto --no-cpu-baseline > gpurun_out/p_c2.json
ncu --set full --clock-control none --import-source on -k regex:k_sweep_g8f -s 20 -c 1 -f -o gpurun_out/prof_r1c_c2 python bench.py --workload c2 --steps 5 --warmup 3 --no-tto --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1
python bench.py --workload c4 --steps 5 --warmup 3 --no-tto --no-cpu-baseline > gpurun_out/p_c4.json
ncu --set full --clock-control none --import-source on -k regex:k_sweep_g8f -s 10 -c 1 -f -o gpurun_out/prof_r1c_c4 python bench.py --workload c4 --steps 5 --warmup 3 --no-tto --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1
echo done

# BCD half-sweeps: DMMA warp-per-row kernel vs the round-1 SIMT kernel
# (MFG_BCD_NO_DMMA=1), plus the BCD parity tests.
export PYTHONDONTWRITEBYTECODE=1
tag=${TAG:-r2c}
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_extras_gpu.py tests/test_sharding.py -x -q -k "bcd or BCD or mf_ or epoch or golden" > gpurun_out/${tag}_pytest_bcd.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_bcd.log
tail -4 gpurun_out/${tag}_pytest_bcd.log
for cfg in "c2 20" "c3 30" "c4 40" ${EXTRA}; do
  set -- $cfg
  echo "== $1 k=$2 DMMA"; timeout 600 python tools/bcd_probe.py $1 $2
  echo "== $1 k=$2 SIMT (round 1)"; MFG_BCD_NO_DMMA=1 timeout 600 python tools/bcd_probe.py $1 $2
done 2>&1 | tee gpurun_out/${tag}_bcd_ab.log

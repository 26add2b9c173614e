# DMMA BCD: cp.async-staged gathers (default) vs register prefetch (MFG_BCD_DM_SYNC=1)
export PYTHONDONTWRITEBYTECODE=1
tag=${TAG:-r2m}
timeout 300 python -m pytest tests/test_kernels_gpu.py tests/test_extras_gpu.py -x -q -k "bcd or BCD or mf_ or epoch or golden" > gpurun_out/${tag}_pytest_bcd.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest_bcd.log
tail -3 gpurun_out/${tag}_pytest_bcd.log
for cfg in "c2 20" "c3 30" "c4 40" ${EXTRA}; do
  set -- $cfg
  echo "== $1 k=$2 async"; timeout 120 python tools/bcd_probe.py $1 $2
  echo "== $1 k=$2 sync"; MFG_BCD_DM_SYNC=1 timeout 120 python tools/bcd_probe.py $1 $2
done 2>&1 | tee gpurun_out/${tag}_bcd_ab.log

export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_extras_gpu.py -x -q > gpurun_out/r2b_pytest_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_pytest_kernels.log
tail -15 gpurun_out/r2b_pytest_kernels.log
WLS="c2 c3 c4" TAG=r2b bash tools/r2_ab_sweep.sh

# GPU parity suite (all -m gpu tests) + compute-sanitizer on the c2-scale kernel tests
set -x
export PYTHONDONTWRITEBYTECODE=1
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu.log
tail -5 gpurun_out/r2_pytest_gpu.log

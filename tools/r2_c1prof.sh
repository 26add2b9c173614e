export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_solver_gpu.py tests/test_c1_gpu.py -x -q -s > gpurun_out/r2i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_pytest.log
tail -3 gpurun_out/r2i_pytest.log; grep "c1 on GPU" gpurun_out/r2i_pytest.log
timeout 600 python tools/kernel_breakdown.py c1 19 > gpurun_out/r2i_c1_breakdown.json 2>&1
head -c 2500 gpurun_out/r2i_c1_breakdown.json

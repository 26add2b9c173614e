# full GPU suite (+ c2 fp32 trace) then the default bench line
export PYTHONDONTWRITEBYTECODE=1
tag=${TAG:-r2h}
timeout 2400 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/${tag}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
tail -4 gpurun_out/${tag}_pytest_gpu.log
grep -h "c1 on GPU\|c2 fp32\|per-iteration" gpurun_out/${tag}_pytest_gpu.log | head
if [ -z "$NOBENCH" ]; then
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -c 3000 gpurun_out/${tag}_bench.json
fi

# one compute-sanitizer tool per call (TOOL=racecheck|synccheck|memcheck)
export PYTHONDONTWRITEBYTECODE=1
python tools/sanitize_probe.py > gpurun_out/r2_san_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool ${TOOL} --print-limit 50 python tools/sanitize_probe.py > gpurun_out/r2_sanitize_${TOOL}.log 2>&1
echo "rc=$?" >> gpurun_out/r2_sanitize_${TOOL}.log
tail -5 gpurun_out/r2_sanitize_${TOOL}.log

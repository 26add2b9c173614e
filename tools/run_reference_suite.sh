# The reference's own test suite (installed with its tests under baseline/_ref,
# see DESIGN.md) with the Omega path routed to libmfg_b200 (GPU box).
REPO=${GRAFT_REPO_ROOT:-$(pwd)}
cd "$REPO/baseline/_ref" || exit 2
PYTHONPATH="$REPO/baseline/_ref:$REPO" PYTHONDONTWRITEBYTECODE=1 timeout 1800 \
  python -m pytest tests -q -p no:cacheprovider -p paper_2204_14067_b200.refplug_pytest ${REF_ARGS} \
  > "$REPO/gpurun_out/${TAG:-r2}_reference_suite.log" 2>&1
echo "rc=$?" >> "$REPO/gpurun_out/${TAG:-r2}_reference_suite.log"
tail -30 "$REPO/gpurun_out/${TAG:-r2}_reference_suite.log"

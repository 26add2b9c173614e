# Installs the unmodified reference into baseline/_ref (git-ignored, shipped to the
# GPU box) together with its own tests, for tests/test_reference_suite_gpu.py.
# Runs in the build container only (/root/reference does not exist on the GPU box).
set -e
REPO=$(cd "$(dirname "$0")/.." && pwd)
[ -d /root/reference/pkg ] || { echo "no /root/reference here"; exit 0; }
rm -rf /tmp/_refpkg && cp -r /root/reference/pkg /tmp/_refpkg
rm -rf "$REPO/baseline/_ref" && mkdir -p "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$REPO/baseline/_ref" /tmp/_refpkg
cp -r /root/reference/pkg/tests "$REPO/baseline/_ref/tests"
ls "$REPO/baseline/_ref"

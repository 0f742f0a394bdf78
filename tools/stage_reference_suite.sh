#!/bin/bash
# Stage the UNMODIFIED reference package and its own test suite under
# baseline/_ref (git-ignored, never committed; it travels to the GPU box with
# the gpurun snapshot) so tools/run_reference_suite.py can run the
# reference's tests against this package on the B200.  Build container only.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/refpkg && cp -r /root/reference/pkg /tmp/refpkg
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" /tmp/refpkg
rm -rf "$ROOT/baseline/_ref/pkg_tests" && cp -r /root/reference/pkg/tests "$ROOT/baseline/_ref/pkg_tests"
echo staged

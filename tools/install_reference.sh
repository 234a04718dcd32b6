#!/bin/bash
# Installs the UNMODIFIED reference package (and its test suite, for
# tests/test_ref_suite.py) into baseline/_ref -- git-ignored, so it never
# enters the repo history, but not gpurun-ignored, so it travels to the GPU
# box.  Run here (where /root/reference exists); offline wheelhouse only.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/kb_refsrc baseline/_ref
cp -r /root/reference/pkg /tmp/kb_refsrc     # the build writes into its source tree
python -m pip install --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target baseline/_ref /tmp/kb_refsrc
mkdir -p baseline/_ref/katzbounds_tests
cp /root/reference/pkg/tests/*.py baseline/_ref/katzbounds_tests/
echo "reference installed: $(ls baseline/_ref)"

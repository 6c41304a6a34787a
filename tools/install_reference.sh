#!/bin/bash
# The one offline install of the reference (rowblock v0.1.0) into baseline/_ref (git-ignored, travels to
# the GPU box with the gpurun snapshot), plus a copy of its own test files for the drop-in shim run
# (tests/test_reference_suite.py).  numpy>=2.0 is already in the image, hence --no-deps; the build
# writes into the source tree, hence the copy under /tmp.  Nothing here enters the repo's history.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/rowblock_src baseline/_ref
cp -r /root/reference/pkg /tmp/rowblock_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse --target baseline/_ref /tmp/rowblock_src
mkdir -p baseline/_ref/ref_tests
cp /root/reference/pkg/tests/*.py baseline/_ref/ref_tests/
cp -r /root/reference/pkg/experiments baseline/_ref/experiments  # A2/A3 read tests/../experiments
printf '[pytest]\n' > baseline/_ref/ref_tests/pytest.ini
echo "installed: $(ls baseline/_ref)"

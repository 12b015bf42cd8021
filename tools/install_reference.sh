#!/bin/sh
# Install the unmodified reference package (undercool) into baseline/_ref (git-ignored,
# shipped to the GPU box with the gpurun snapshot).  Used by
# tests/test_gpu_reference_driver.py (the reference's own simulate() with the
# drop-in substituted) and bench.py --impl reference (its single-core timing).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/uc_refcopy baseline/_ref
cp -r /root/reference/pkg /tmp/uc_refcopy   # the build writes into the source tree
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/uc_refcopy

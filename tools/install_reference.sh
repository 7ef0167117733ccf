#!/bin/bash
# The one offline install of the reference (base contract): mlower from
# /root/reference into baseline/_ref (git-ignored; it travels to the GPU box
# with the snapshot).  The reference's own test suite is placed beside it
# (baseline/_ref/mlower_tests) so tests/test_gpu_reference_swap.py can run the
# reference's tests with its executor swapped for ours on the B200.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/mlower_src baseline/_ref
cp -r /root/reference/pkg /tmp/mlower_src    # the build writes into the source tree; /root/reference is read-only
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
  --target baseline/_ref /tmp/mlower_src
cp -r /root/reference/pkg/tests baseline/_ref/mlower_tests
cp -r /root/reference/pkg/exporter baseline/_ref/mlower_exporter
echo "installed: $(ls baseline/_ref)"

#!/bin/bash
# Install the unmodified reference package into baseline/_ref (git-ignored,
# travels to the GPU box with gpurun) so the integration tests can import it
# there; its test files are placed beside it (baseline/_ref/topofuse_tests)
# for tests/test_gpu_integration.py to run against the B200 kernels.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/refpkg && cp -r /root/reference/pkg /tmp/refpkg
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/refpkg --no-deps --upgrade
rm -rf baseline/_ref/topofuse_tests && cp -r /root/reference/pkg/tests baseline/_ref/topofuse_tests
echo "installed: $(ls baseline/_ref)"

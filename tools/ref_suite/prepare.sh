#!/usr/bin/env bash
# Run HERE (the build container; /root/reference exists only here): install
# the unmodified reference package into baseline/_ref (git-ignored, travels to
# the GPU box with the gpurun snapshot) and stage its test suite next to it.
set -e
cd "$(dirname "$0")/../.."
rm -rf /tmp/bltc_refpkg baseline/_ref
cp -r /root/reference/pkg /tmp/bltc_refpkg
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target baseline/_ref /tmp/bltc_refpkg
cp -r /root/reference/pkg/tests baseline/_ref/_tests
echo "reference installed in baseline/_ref, tests in baseline/_ref/_tests"

#!/bin/bash
# Stage the reference for the GPU box (build container only; /root/reference
# does not exist there).  Both targets are git-ignored and travel with the
# gpurun snapshot:
#   baseline/_ref        -- the reference package, pip-installed (bench.py --impl reference)
#   baseline/_ref_tests  -- the reference's own test suite (tools/reference_suite.py)
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/meshplan_ref_src && cp -r /root/reference/pkg /tmp/meshplan_ref_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref --upgrade /tmp/meshplan_ref_src > /dev/null
rm -rf baseline/_ref_tests && cp -r /root/reference/pkg/tests baseline/_ref_tests
echo "staged baseline/_ref and baseline/_ref_tests"

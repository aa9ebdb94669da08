#!/bin/bash
# Stage the reference's own test suite next to the installed reference
# package (git-ignored, travels to the GPU box with the gpurun snapshot) so
# tests/test_conformance.py can run it there.  Nothing is committed.
set -e
cd "$(dirname "$0")/.."
rm -rf baseline/_ref_tests
mkdir -p baseline
cp -r /root/reference/pkg/tests baseline/_ref_tests
echo "staged $(ls baseline/_ref_tests | wc -l) files into baseline/_ref_tests"

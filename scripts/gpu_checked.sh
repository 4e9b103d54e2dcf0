#!/bin/bash
# The GPU test suite against the CHECKED build (libtwc_checked.so: device-side asserts on every
# ring / staging index, computed global index and capacity; build.py), the replacement for
# compute-sanitizer, which this GPU pool does not allow.  A violated assert fails the test with
# "Assertion ... failed" (file and line) in the log.  usage: bash scripts/gpu_checked.sh TAG
TAG=${1:-checked}
mkdir -p gpurun_out
python -m paper_2412_12382_b200.build --checked > /dev/null || exit 1
TWC_LIB=checked timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider \
    > gpurun_out/pytest_${TAG}_checked.log 2>&1
rc=$?; echo checked_pytest_exit=$rc; tail -5 gpurun_out/pytest_${TAG}_checked.log
grep -c "Assertion" gpurun_out/pytest_${TAG}_checked.log
exit $rc

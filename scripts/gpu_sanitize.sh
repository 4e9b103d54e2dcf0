#!/bin/bash
# compute-sanitizer over one small pass of every kernel family (scripts/sanitize_run.py):
# memcheck (out-of-bounds / misaligned accesses, leaks), racecheck (shared-memory hazards: K2's
# warp-synchronous rings, the union-find is global memory), synccheck (illegal barriers /
# __syncwarp masks), initcheck (reads of uninitialised device memory).  Logs in gpurun_out/.
TAG=${1:-san}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python scripts/sanitize_run.py > gpurun_out/sanitizer_${TAG}_${tool}.log 2>&1
  echo "$tool exit=$?"
  tail -4 gpurun_out/sanitizer_${TAG}_${tool}.log
done

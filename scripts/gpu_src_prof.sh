#!/bin/bash
# Per-source-line instruction counts of one kernel for each value of a variant env var.
# usage: bash scripts/gpu_src_prof.sh TAG VAR "v0 v1" KERNEL_REGEX
TAG=$1; VAR=$2; VALS=$3; KRE=$4
mkdir -p gpurun_out
for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1 || exit 1
  env $VAR=$v timeout 600 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section Occupancy \
      --metrics smsp__inst_executed.sum,gpu__time_duration.sum \
      --clock-control none --import-source on -k regex:"$KRE" -s 2 -c 1 -o gpurun_out/src_${TAG}_$v \
      python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/src_${TAG}_$v.log 2>&1
  echo ncu_$v=$?
done

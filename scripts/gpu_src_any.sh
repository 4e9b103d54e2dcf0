#!/bin/bash
# ncu --set full + SASS source page of one kernel on one bench config.
# usage: bash scripts/gpu_src_any.sh TAG KERNEL_REGEX CONFIG [SKIP]
TAG=$1; KRE=$2; CFG=${3:-5}; SKIP=${4:-1}
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_${TAG}.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE}" \
    -s ${SKIP} -c 1 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo ncu_exit=$?
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${TAG}.csv 2>/dev/null
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}.csv 2>/dev/null
rm -f gpurun_out/prof_${TAG}.ncu-rep

#!/bin/bash
# One ncu --set full capture of K2 with source, exported on the box as the SASS-level source page
# (per-instruction executed counts, stall samples, shared / global wavefronts).
# usage: bash scripts/gpu_src_k2.sh TAG [KERNEL_REGEX]
TAG=${1:-srck2}; KRE=${2:-k2_intersect}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_${TAG}.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE}" \
    -s 2 -c 1 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo ncu_exit=$?
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${TAG}.csv 2>/dev/null
ncu -i gpurun_out/prof_${TAG}.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}.csv 2>/dev/null
rm -f gpurun_out/prof_${TAG}.ncu-rep
ls -la gpurun_out | tail -5

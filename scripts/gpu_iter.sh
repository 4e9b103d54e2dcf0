#!/bin/bash
# One GPU iteration: parity tests, bench (JSON line), launch list and one ncu --set full capture.
# usage: bash scripts/gpu_iter.sh TAG [KERNEL_REGEX] [SKIP] [COUNT]
TAG=${1:-iter}
KRE=${2:-"k1_count|k1_scatter|k2_intersect|k3_score|k_band_count|k_band_scatter|k_hook_list"}
SKIP=${3:-4}
CNT=${4:-8}
mkdir -p gpurun_out
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo pytest_exit=$?
tail -5 gpurun_out/pytest_${TAG}.log
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo bench_exit=$?
cat gpurun_out/bench_${TAG}.json
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1; echo ncu1_exit=$?
ncu --set full --clock-control none --import-source on -k regex:"${KRE}" -s ${SKIP} -c ${CNT} -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1; echo ncu2_exit=$?

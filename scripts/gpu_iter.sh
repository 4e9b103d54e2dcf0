#!/bin/bash
# One GPU iteration: parity tests, bench (JSON line), launch list and one ncu --set full capture.
# Every step is wrapped in its own timeout and the later steps only run if the earlier ones
# exited 0 (ncu only profiles a command that has just run cleanly without it).
# usage: bash scripts/gpu_iter.sh TAG [KERNEL_REGEX] [SKIP] [COUNT]
TAG=${1:-iter}
KRE=${2:-"k1_bits|k1_write|k2_intersect|k3_score|k_band_place|k_hook_list|k_finalize|k_part_edges"}
SKIP=${3:-3}
CNT=${4:-8}
mkdir -p gpurun_out
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1
rc=$?; echo pytest_exit=$rc
tail -5 gpurun_out/pytest_${TAG}.log
[ $rc -eq 0 ] || exit $rc
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
rc=$?; echo bench_exit=$rc
cat gpurun_out/bench_${TAG}.json
[ $rc -eq 0 ] || exit $rc
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_${TAG}.log 2>&1
rc=$?; echo plain_exit=$rc
[ $rc -eq 0 ] || exit $rc
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
echo ncu1_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE}" \
    -s ${SKIP} -c ${CNT} -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo ncu2_exit=$?

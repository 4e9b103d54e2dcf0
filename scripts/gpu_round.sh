#!/bin/bash
# Full GPU pass: gpu tests, sanitizers, then bench + launch list + ncu --set full of the step's
# kernels (scripts/gpu_iter.sh without its pytest).  usage: bash scripts/gpu_round.sh TAG
TAG=${1:-round}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1
rc=$?; echo pytest_exit=$rc; tail -5 gpurun_out/pytest_${TAG}.log
bash scripts/gpu_sanitize.sh $TAG
[ $rc -eq 0 ] || exit $rc
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
rc=$?; echo bench_exit=$rc; tail -c 600 gpurun_out/bench_${TAG}.json
[ $rc -eq 0 ] || exit $rc
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_${TAG}.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
echo ncu1_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k1_bits|k1_write|k2_intersect|k3_score|k_band_place|k_hook_list|k_finalize" \
    -s 3 -c 7 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo ncu2_exit=$?

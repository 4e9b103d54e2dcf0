#!/bin/bash
# Round-2 final check of HEAD: full GPU suite, bench, launch list, one --set full capture
# (K1/K2/K3 with source), the source page of K2 exported as CSV on the box.
TAG=${1:-r2k}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1
rc=$?; echo pytest_exit=$rc; tail -3 gpurun_out/pytest_${TAG}.log
[ $rc -eq 0 ] || exit $rc
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo bench_exit=$?; head -c 600 gpurun_out/bench_${TAG}.json; echo
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_${TAG}.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
echo ncu1_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k1_bits|k1_write|k2_intersect|k3_score|k_band_place|k_hook_list|k_finalize" \
    -s 3 -c 7 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo ncu2_exit=$?
ncu -i gpurun_out/prof_${TAG}.ncu-rep -k regex:k2_intersect --page source --csv --print-source sass > gpurun_out/src_k2_${TAG}.csv 2>/dev/null
ncu -i gpurun_out/prof_${TAG}.ncu-rep -k regex:k3_score --page source --csv --print-source sass > gpurun_out/src_k3_${TAG}.csv 2>/dev/null
ncu -i gpurun_out/prof_${TAG}.ncu-rep -k regex:k1_bits --page source --csv --print-source sass > gpurun_out/src_k1_${TAG}.csv 2>/dev/null
ls -la gpurun_out | tail -20

#!/bin/bash
# Round-2 final measurement of HEAD: full GPU suite (normal and checked build), launch list and
# ncu --set full capture summarised ON THE BOX (so the bench line that follows cites the ncu
# capture of the same gpurun in roofline.traffic_source), bench lines for configs 5 and 1-4,
# R-MAT / NEXT / distributed-emulation measurements.
TAG=${1:-r2l}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1
rc=$?; echo pytest_exit=$rc; tail -3 gpurun_out/pytest_${TAG}.log
[ $rc -eq 0 ] || exit $rc
TWC_LIB=checked timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider \
    > gpurun_out/pytest_${TAG}_checked.log 2>&1
echo checked_exit=$? assertions=$(grep -c "Assertion" gpurun_out/pytest_${TAG}_checked.log)
tail -2 gpurun_out/pytest_${TAG}_checked.log
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_${TAG}.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
echo ncu1_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k1_bits|k1_write|k2_intersect|k3_score|k_band_place|k_hook_list|k_finalize" \
    -s 3 -c 7 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo ncu2_exit=$?
python scripts/summarize_ncu.py ${TAG} gpurun_out/prof_${TAG}.ncu-rep gpurun_out/launches_${TAG}.csv
ncu -i gpurun_out/prof_${TAG}.ncu-rep -k regex:k2_intersect --page source --csv --print-source sass > gpurun_out/src_k2_${TAG}.csv 2>/dev/null
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo bench_exit=$?; head -c 400 gpurun_out/bench_${TAG}.json; echo
cp gpurun_out/bench_${TAG}.json profiles/${TAG}_bench.json
mkdir -p profiles/${TAG}_configs
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 40 --warmup 5 > profiles/${TAG}_configs/bench_cfg$c.json 2> gpurun_out/bench_${TAG}_cfg$c.err
  echo cfg$c exit=$?
done
timeout 1800 python scripts/bench_rmat.py --tag ${TAG} > gpurun_out/rmat_${TAG}.log 2>&1; echo rmat_exit=$?
timeout 1200 python scripts/bench_next.py --tag ${TAG} > gpurun_out/next_${TAG}.log 2>&1; echo next_exit=$?
timeout 1200 python scripts/bench_dist_emulated.py > gpurun_out/dist_${TAG}.log 2>&1; echo dist_exit=$?
rm -f gpurun_out/prof_${TAG}.ncu-rep.tmp
mkdir -p gpurun_out/profiles_${TAG}; cp -r profiles/${TAG}_* profiles/k2_ncu_summary.json profiles/rmat_${TAG}.json profiles/next_${TAG}.json profiles/dist_emulated*.json gpurun_out/profiles_${TAG}/ 2>/dev/null
tail -8 gpurun_out/rmat_${TAG}.log; tail -4 gpurun_out/dist_${TAG}.log

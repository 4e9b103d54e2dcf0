#!/bin/bash
# A/B of kernel variants selected by an environment variable of the library (same build):
# parity tests under the new default, then the kernel-only bench per value, then a short ncu
# pass on the chosen kernel per value.
# usage: bash scripts/gpu_ab_env.sh TAG VAR "v0 v1 ..." [KERNEL_REGEX] [PYTEST_TARGET]
TAG=$1; VAR=$2; VALS=$3; KRE=${4:-k2_intersect}; PT=${5:-tests/test_gpu_parity.py}
mkdir -p gpurun_out
if [ "$PT" != none ]; then
  timeout 900 python -m pytest $PT -x -q > gpurun_out/pytest_${TAG}.log 2>&1
  rc=$?; echo pytest_exit=$rc; tail -3 gpurun_out/pytest_${TAG}.log
  [ $rc -eq 0 ] || exit $rc
fi
for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/ab_${TAG}_$v.json 2> gpurun_out/ab_${TAG}_$v.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab_${TAG}_$v.json').read().strip().splitlines()[-1]);print('$VAR=$v', round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['phases_ms'].items()}, d['clocks'])"
done
for v in $VALS; do
  env $VAR=$v timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
      --clock-control none -k regex:"$KRE" -s 2 -c 1 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
      > gpurun_out/ncu_${TAG}_$v.csv 2>/dev/null
  echo "== $VAR=$v"; grep -E '"(gpu__time|smsp__inst|smsp__issue|dram__bytes|sm__warps)' gpurun_out/ncu_${TAG}_$v.csv | awk -F'","' '{print $(NF-2), $NF}'
done

#!/bin/bash
# A/B of library variants selected by an environment variable (same build): per value, the
# parity tests under that value, the kernel-only bench line, and a short ncu pass on the
# kernel(s) of interest.
# usage: bash scripts/gpu_ab_vars.sh TAG VAR "v0 v1 ..." [KERNEL_REGEX] [PYTEST_FILE|none] [-k EXPR]
TAG=$1; VAR=$2; VALS=$3; KRE=${4:-k2_intersect}; PT=${5:-tests/test_gpu_parity.py}; KX=${6:-}
mkdir -p gpurun_out
for v in $VALS; do
  if [ "$PT" != none ]; then
    if [ -n "$KX" ]; then
      env $VAR=$v timeout 900 python -m pytest $PT -x -q -k "$KX" > gpurun_out/pytest_${TAG}_$v.log 2>&1
    else
      env $VAR=$v timeout 900 python -m pytest $PT -x -q > gpurun_out/pytest_${TAG}_$v.log 2>&1
    fi
    rc=$?; echo "$VAR=$v pytest_exit=$rc"; tail -2 gpurun_out/pytest_${TAG}_$v.log
    [ $rc -eq 0 ] || continue
  fi
  env $VAR=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/ab_${TAG}_$v.json 2> gpurun_out/ab_${TAG}_$v.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab_${TAG}_$v.json').read().strip().splitlines()[-1]);print('$VAR=$v', round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['phases_ms'].items()}, d['clocks'].get('sm_mhz'))"
done
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
for v in $VALS; do
  env $VAR=$v timeout 300 ncu --metrics $M --clock-control none -k regex:"$KRE" -s 2 -c 1 --csv \
      python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG}_$v.csv 2>/dev/null
  echo "== $VAR=$v"; grep -E '^"[0-9]' gpurun_out/ncu_${TAG}_$v.csv | awk -F'","' '{print $(NF-2), $NF}'
done

#!/bin/bash
# A/B of library variants selected by environment variables (same build).  Every argument after
# the options is one variant: a quoted list of VAR=value assignments ("" = defaults).
#   -p FILE   parity tests run under the FIRST variant(s) listed in -P (default: none)
#   -k REGEX  kernels for the short ncu pass (default k2_intersect), -n N ncu launches to take
# usage: bash scripts/gpu_ab_env2.sh TAG [-t "pytest args"] [-k REGEX] [-c COUNT] [-N "idx idx"] -- "A=1 B=2" "A=3" ...
TAG=$1; shift
PT=""; KRE=k2_intersect; CNT=1; NIDX=""
while [ "$1" != "--" ]; do
  case $1 in
    -t) PT=$2; shift 2;;
    -k) KRE=$2; shift 2;;
    -c) CNT=$2; shift 2;;
    -N) NIDX=$2; shift 2;;
    *) echo "bad option $1"; exit 2;;
  esac
done
shift
mkdir -p gpurun_out
i=0
for v in "$@"; do
  if [ -n "$PT" ]; then
    env $v timeout 1200 python -m pytest $PT -x -q > gpurun_out/pytest_${TAG}_$i.log 2>&1
    rc=$?; echo "[$i] $v pytest_exit=$rc"; tail -2 gpurun_out/pytest_${TAG}_$i.log
    [ $rc -eq 0 ] || { i=$((i+1)); continue; }
  fi
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/ab_${TAG}_$i.json 2> gpurun_out/ab_${TAG}_$i.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab_${TAG}_$i.json').read().strip().splitlines()[-1]);print('[$i] $v', round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['phases_ms'].items()}, d['clocks'].get('sm_mhz'))"
  i=$((i+1))
done
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,sm__warps_active.avg.pct_of_peak_sustained_active
i=0
for v in "$@"; do
  if [ -z "$NIDX" ] || [[ " $NIDX " == *" $i "* ]]; then
    env $v timeout 300 ncu --metrics $M --clock-control none -k regex:"$KRE" -s $((2*CNT)) -c $CNT --csv \
        python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG}_$i.csv 2>/dev/null
    echo "== [$i] $v"; grep -E '^"[0-9]' gpurun_out/ncu_${TAG}_$i.csv | awk -F'","' '{print substr($5,1,28), $(NF-2), $NF}'
  fi
  i=$((i+1))
done

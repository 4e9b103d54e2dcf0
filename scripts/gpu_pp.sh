#!/bin/bash
# A/B: K2 filter probes predicated on the entry's validity (TWC_LIB=pp, -DTWC_K2_PREDPROBE)
mkdir -p gpurun_out
run() {
  TWC_LIB=$1 timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_pp.json 2> gpurun_out/ab_pp.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab_pp.json').read().strip().splitlines()[-1]);print('lib=$1', round(d['ms_per_step'],4), {k: round(v, 3) for k, v in d['phases_ms'].items()})"
}
run ""; run pp; run ""; run pp
TWC_LIB=pp timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
for lib in "" pp; do
  TWC_LIB=$lib timeout 600 ncu --clock-control none \
      --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum \
      -k regex:"k2_intersect" -s 1 -c 1 --csv --log-file gpurun_out/ncu_pp_$lib.csv $CMD > /dev/null 2>&1
  echo "lib=$lib"; grep -E "k2_intersect" gpurun_out/ncu_pp_$lib.csv | awk -F'","' '{print $(NF-2), $(NF)}'
done

#!/bin/bash
# A/B: K3 reading rp_or[v], rp_or[v+1] (16 MB, own persisting window) instead of vinfo[v] (TWC_LIB=rpor)
mkdir -p gpurun_out
run() {
  TWC_LIB=$1 timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_rpor.json 2> gpurun_out/ab_rpor.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab_rpor.json').read().strip().splitlines()[-1]);print('lib=$1', round(d['ms_per_step'],4), {k: round(v, 3) for k, v in d['phases_ms'].items()}, (d.get('cuda_graph') or {}).get('ms_per_step'))"
}
run ""; run rpor; run ""; run rpor
TWC_LIB=rpor timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
for lib in "" rpor; do
  TWC_LIB=$lib timeout 600 ncu --cache-control none --clock-control none \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct \
      -k regex:"k3_score" -s 1 -c 1 --csv --log-file gpurun_out/ncu_rpor_$lib.csv $CMD > /dev/null 2>&1
  echo "lib=$lib"; grep -E "k3_score" gpurun_out/ncu_rpor_$lib.csv | awk -F'","' '{print $(NF-2), $(NF)}'
done

#!/bin/bash
# quick check of the default-on adaptive L2 window: config 5 / 4 bench lines, similarity timings + parity
mkdir -p gpurun_out
for c in 5 4 5; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_l2r.json 2> gpurun_out/ab_l2r.err
  python -c "
import json;d=json.loads(open('gpurun_out/ab_l2r.json').read().strip().splitlines()[-1]);print('cfg$c', round(d['ms_per_step'],4), {k: round(v, 3) for k, v in d['phases_ms'].items()}, (d.get('cuda_graph') or {}).get('ms_per_step'))"
done
TWC_L2_PERSIST_MB=0 timeout 300 python bench.py --config 4 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_l2r.json 2> gpurun_out/ab_l2r.err
python -c "
import json;d=json.loads(open('gpurun_out/ab_l2r.json').read().strip().splitlines()[-1]);print('cfg4 off', round(d['ms_per_step'],4))"
timeout 900 python -m pytest tests/test_gpu_similarity.py -x -q 2>&1 | tail -2
timeout 600 python scripts/bench_next.py --tag l2r --graphs 5 --no-oracle 2>&1 | grep similarity | cut -c1-120

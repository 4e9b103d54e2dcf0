#!/bin/bash
# A/B: run the kernel-only bench with alternative builds of libtwc.so (scripts/ab/lib*.so)
mkdir -p gpurun_out
for lib in "$@"; do
  cp scripts/ab/$lib paper_2412_12382_b200/libtwc.so
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab_$lib.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab_$lib.json').read().strip().splitlines()[-1]);print('$lib', round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['phases_ms'].items()})"
done

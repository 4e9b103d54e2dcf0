#!/bin/bash
# A/B of the persisting-L2 window: set-aside size x (vinfo only | window moved per phase)
TAG=${1:-l2q}
mkdir -p gpurun_out
run() {  # mb phases config steps
  TWC_L2_PERSIST_MB=$1 TWC_L2_PHASES=$2 timeout 300 python bench.py --config $3 --steps $4 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/ab_${TAG}.json 2> gpurun_out/ab_${TAG}.err
  python - <<PY
import json
d = json.loads(open("gpurun_out/ab_${TAG}.json").read().strip().splitlines()[-1])
g = d.get("cuda_graph") or {}
print("cfg$3 mb=$1 phases=$2 step %.4f" % d["ms_per_step"], {k: round(v, 3) for k, v in d["phases_ms"].items()}, "graph", round(g.get("ms_per_step", 0), 4))
PY
}
for rep in 1 2; do
  run 0 0 5 30; run 32 0 5 30; run 32 1 5 30; run 24 0 5 30; run 24 1 5 30; run 16 1 5 30; run 40 1 5 30
done
for c in 2 3 4; do run 0 0 $c 60; run 32 0 $c 60; run 32 1 $c 60; run 0 0 $c 60; run 32 1 $c 60; done
TWC_L2_PERSIST_MB=32 TWC_L2_PHASES=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_${TAG}_par.log 2>&1
echo parity_exit=$?; tail -2 gpurun_out/pytest_${TAG}_par.log

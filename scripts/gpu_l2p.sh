#!/bin/bash
# A/B of the persisting-L2 window on vinfo (TWC_L2_PERSIST_MB, twc_api.cu) and check of the new
# k_similarity: similarity parity, kernel-only bench lines per set-aside size, K3 / K2 DRAM bytes
# under ncu with the caches left alone, parity (incl. the CUDA-graph replay) with the window on.
TAG=${1:-l2p}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_similarity.py -x -q > gpurun_out/pytest_${TAG}_sim.log 2>&1
echo sim_exit=$?; tail -2 gpurun_out/pytest_${TAG}_sim.log
for mb in 0 32 48 64 0 32; do
  TWC_L2_PERSIST_MB=$mb timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/ab_${TAG}_$mb.json 2> gpurun_out/ab_${TAG}_$mb.err
  python - <<PY
import json
d = json.loads(open("gpurun_out/ab_${TAG}_$mb.json").read().strip().splitlines()[-1])
print("mb=$mb step %.3f" % d["ms_per_step"], {k: round(v, 3) for k, v in d["phases_ms"].items()},
      "graph", round(d.get("cuda_graph", {}).get("ms_per_step", 0), 3) if isinstance(d.get("cuda_graph"), dict) else d.get("cuda_graph"))
PY
done
for c in 2 4; do for mb in 0 32; do
  TWC_L2_PERSIST_MB=$mb timeout 300 python bench.py --config $c --steps 40 --warmup 5 --no-e2e --no-cpu-baseline \
      > gpurun_out/ab_${TAG}_c${c}_$mb.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab_${TAG}_c${c}_$mb.json').read().strip().splitlines()[-1]);print('cfg$c mb=$mb', round(d['ms_per_step'],4))"
done; done
TWC_L2_PERSIST_MB=32 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_${TAG}_par.log 2>&1
echo parity_exit=$?; tail -2 gpurun_out/pytest_${TAG}_par.log
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
for mb in 0 32; do
  TWC_L2_PERSIST_MB=$mb timeout 600 ncu --cache-control none --clock-control none \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
      -k regex:"k2_intersect|k3_score" -s 2 -c 2 --csv --log-file gpurun_out/ncu_${TAG}_$mb.csv $CMD > /dev/null 2>&1
  echo ncu_$mb exit=$?; grep -E "k2_intersect|k3_score" gpurun_out/ncu_${TAG}_$mb.csv | awk -F'","' '{print $5, $(NF-2), $(NF)}' | cut -c1-160
done
timeout 600 python scripts/bench_next.py --tag ${TAG} --graphs 5 --no-oracle > gpurun_out/next_${TAG}.log 2>&1
grep similarity gpurun_out/next_${TAG}.log | cut -c1-200

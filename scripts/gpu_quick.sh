#!/bin/bash
# Quick A/B iteration on one GPU: the parity tests (config 5 full size included) and a
# kernel-only bench line.  usage: bash scripts/gpu_quick.sh TAG
TAG=${1:-quick}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_${TAG}.log 2>&1
rc=$?; echo pytest_exit=$rc; tail -3 gpurun_out/pytest_${TAG}.log
[ $rc -eq 0 ] || exit $rc
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
    > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
rc=$?; echo bench_exit=$rc
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_${TAG}.json").read().strip().splitlines()[-1])
print("value %.3e ms %.3f" % (d["value"], d["ms_per_step"]))
print("phases", {k: round(v, 3) for k, v in d["phases_ms"].items()})
print("separate", {k: round(v, 3) for k, v in d["separate_calls_ms"].items()})
print("selection", d.get("selection"))
print("frac %.3f clocks %s" % (d["roofline"]["frac"], d["clocks"]))
PY

mkdir -p gpurun_out
TAG=$1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config_parity_full_size or fused or hub or random or dense" > gpurun_out/pytest_${TAG}.log 2>&1
rc=$?; echo pytest_exit=$rc; tail -1 gpurun_out/pytest_${TAG}.log
[ $rc -eq 0 ] || exit $rc
for i in 1 2; do
timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_$i.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/bench_${TAG}_$i.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['phases_ms'].items()})"
done
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none -k regex:"k2_intersect" -s 2 -c 1 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG}.csv 2>/dev/null
grep -E '^"[0-9]' gpurun_out/ncu_${TAG}.csv | awk -F'","' '{print $(NF-2), $NF}'

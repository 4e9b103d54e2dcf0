set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r1_a.json 2> gpurun_out/bench_r1_a.err; echo bench_exit=$?
tail -c 3000 gpurun_out/bench_r1_a.json
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo ncu1_exit=$?
ncu --set full --clock-control none --import-source on -k regex:"k2_intersect|k3_score|k_hook_band|k1_count|k1_scatter|k_finalize" -s 11 -c 8 -o gpurun_out/prof_r1 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2_exit=$?
ls -la gpurun_out

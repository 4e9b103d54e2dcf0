mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_stats.py -x -q > gpurun_out/pytest_r2g.log 2>&1
rc=$?; echo pytest_exit=$rc; tail -2 gpurun_out/pytest_r2g.log
[ $rc -eq 0 ] || exit $rc
timeout 600 python bench.py > gpurun_out/bench_r2g.json 2> gpurun_out/bench_r2g.err
echo bench_exit=$?
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_r2g.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_r2g.csv $CMD > gpurun_out/ncu_launches_r2g.log 2>&1
echo ncu1_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k1_bits|k1_write|k2_intersect|k3_score|k_band_place|k_hook_list|k_finalize" \
    -s 3 -c 7 -o gpurun_out/prof_r2g $CMD > gpurun_out/ncu_full_r2g.log 2>&1
echo ncu2_exit=$?

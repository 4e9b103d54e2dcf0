mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2i.log 2>&1
rc=$?; echo pytest_exit=$rc; tail -2 gpurun_out/pytest_r2i.log
[ $rc -eq 0 ] || exit $rc
timeout 600 python bench.py > gpurun_out/bench_r2i.json 2> gpurun_out/bench_r2i.err
echo bench_exit=$?
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_r2i.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_r2i.csv $CMD > gpurun_out/ncu_launches_r2i.log 2>&1
echo ncu1_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k1_bits|k1_write|k2_intersect|k3_score|k_band_place|k_hook_list|k_finalize" \
    -s 3 -c 7 -o gpurun_out/prof_r2i $CMD > gpurun_out/ncu_full_r2i.log 2>&1
echo ncu2_exit=$?
bash scripts/gpu_checked.sh r2i

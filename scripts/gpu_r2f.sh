mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q > gpurun_out/pytest_r2f.log 2>&1
echo pytest_exit=$?; tail -2 gpurun_out/pytest_r2f.log
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 40 --warmup 5 > gpurun_out/bench_r2f_cfg$c.json 2> gpurun_out/bench_r2f_cfg$c.err
  echo cfg$c exit=$?
done
timeout 1800 python scripts/oracle_baseline.py --out gpurun_out/oracle_baseline_r2 > gpurun_out/oracle_baseline_r2.log 2>&1
echo oracle_exit=$?; tail -3 gpurun_out/oracle_baseline_r2.log

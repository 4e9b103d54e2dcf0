mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_r2c_dist.log 2>&1
echo dist_pytest_exit=$?; tail -15 gpurun_out/pytest_r2c_dist.log
timeout 900 python scripts/bench_dist_emulated.py --config 5 --worlds 1,2,4,8 --reps 3 > gpurun_out/dist_emul_r2c.json 2> gpurun_out/dist_emul_r2c.err
echo emul_exit=$?; tail -5 gpurun_out/dist_emul_r2c.err
bash scripts/gpu_ab_vars.sh k2b TWC_K2 "13,5 14,5 15,3 13,6"

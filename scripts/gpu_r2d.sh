mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_r2d_dist.log 2>&1
echo dist_pytest_exit=$?; tail -3 gpurun_out/pytest_r2d_dist.log
timeout 900 python scripts/bench_dist_emulated.py --config 5 --worlds 1,2,4,8 --reps 3 > gpurun_out/dist_emul_r2d.json 2> gpurun_out/dist_emul_r2d.err
echo emul_exit=$?; tail -5 gpurun_out/dist_emul_r2d.err
bash scripts/gpu_ab_vars.sh k2c TWC_K2 "256 64 128"
bash scripts/gpu_checked.sh r2d

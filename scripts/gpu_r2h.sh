mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py tests/test_gpu_k4.py -x -q > gpurun_out/pytest_r2h.log 2>&1
rc=$?; echo pytest_exit=$rc; tail -2 gpurun_out/pytest_r2h.log
[ $rc -eq 0 ] || exit $rc
timeout 1800 python scripts/bench_rmat.py --tag r2h > gpurun_out/rmat_r2h.log 2>&1; echo rmat_exit=$?
cp profiles/rmat_r2h.json gpurun_out/ 2>/dev/null
timeout 1200 python scripts/bench_next.py --tag r2h > gpurun_out/next_r2h.log 2>&1; echo next_exit=$?
cp profiles/next_r2h.json gpurun_out/ 2>/dev/null
tail -12 gpurun_out/rmat_r2h.log; tail -12 gpurun_out/next_r2h.log

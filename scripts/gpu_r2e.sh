mkdir -p gpurun_out
# bench N>1 code path (functional: 2 ranks on cuda:0 over gloo)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 1 --backend gloo --same-device > gpurun_out/bench_r2e_n2gloo.json 2> gpurun_out/bench_r2e_n2gloo.err
echo n2_exit=$?; tail -c 1500 gpurun_out/bench_r2e_n2gloo.json; tail -3 gpurun_out/bench_r2e_n2gloo.err
bash scripts/gpu_ab_vars.sh k2d TWC_K2 "256,13,128,5 256,13,64,5 256,12,64,5 256,12,64,6" k2_intersect none
bash scripts/gpu_ab_vars.sh k3a TWC_K3 "0 1 2 3" k3_score none

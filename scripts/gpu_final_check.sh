#!/bin/bash
# round-end sanity on the GPU box: smoke(), the reference arm, a 2-rank same-device run of the
# distributed step (code path only, not a measurement), default bench line
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" 2>&1 | tail -3
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_final.json 2> gpurun_out/ref_final.err
echo ref_exit=$?; tail -c 700 gpurun_out/ref_final.json; echo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus 2 --steps 3 --warmup 1 --backend gloo --same-device > gpurun_out/bs_final.json 2> gpurun_out/bs_final.err
echo dist_exit=$?; tail -c 500 gpurun_out/bs_final.json; echo

#!/bin/bash
mkdir -p gpurun_out/r02m
(timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) > gpurun_out/r02m/n1_cfg5.json
for c in 1 4; do
(RB_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config $c --steps 5 --warmup 3 --e2e-steps 2 2>&1 | tail -3) > gpurun_out/r02m/n2_cfg$c.log
done

#!/bin/bash
mkdir -p gpurun_out/r02sh
for c in 5 2 4 3; do timeout 900 python tools/shard_sim.py $c 2,4,8 10 2>&1 | tail -1 >> gpurun_out/r02sh/proj.jsonl; done

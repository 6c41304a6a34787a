#!/bin/bash
# Re-bench the CUDA-core configs after the CSR gather engine's 4-CTA/SM build.
mkdir -p gpurun_out/r02c
for c in 1 2b 3; do
  (timeout 900 python bench.py --config $c --steps 30 --warmup 5 --cpu-seconds 8 2>gpurun_out/r02c/cfg$c.err | tail -1) > gpurun_out/r02c/cfg$c.json
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02c/launches_cfg3.csv python tools/spmm_once.py 3 1 3 > gpurun_out/r02c/ll3.log 2>&1

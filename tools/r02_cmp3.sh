#!/bin/bash
mkdir -p gpurun_out/r02c
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02c/ll_cfg3.csv python tools/spmm_once.py 3 1 3 > gpurun_out/r02c/ll3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02c/ll_cfg2b.csv python tools/spmm_once.py 2b 1 3 > gpurun_out/r02c/ll2b.log 2>&1
for c in 1 2b 3; do (timeout 600 python bench.py --config $c --steps 30 --warmup 5 --cpu-seconds 5 2>&1 | tail -1) > gpurun_out/r02c/final_b$c.json; done

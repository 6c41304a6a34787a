#!/bin/bash
mkdir -p gpurun_out/r02s gpurun_out/r02p
(timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or medium or shapes or shard" 2>&1 | tail -5) > gpurun_out/r02s/tests.log
RB_SWEEP_DELAY=16 ROWBLOCK_B200_LIB=variants/noload.so timeout 300 python tools/spmm_once.py 5 1 2 > gpurun_out/r02p/noload.log 2>&1
RB_SWEEP_DELAY=16 ROWBLOCK_B200_LIB=variants/prof.so timeout 300 python tools/spmm_once.py 5 1 2 > gpurun_out/r02p/prof_d16.log 2>&1
for d in 8 16 32; do (RB_SWEEP_DELAY=$d timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) > gpurun_out/r02s/bench5_d$d.json; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_sweep -s 2 -c 1 -o gpurun_out/r02s/ncu_sweep_cfg5 -f python tools/spmm_once.py 5 1 3 > gpurun_out/r02s/ncu.log 2>&1

#!/bin/bash
mkdir -p gpurun_out/r02s gpurun_out/r02p
(timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or medium" 2>&1 | tail -3) > gpurun_out/r02s/tests.log
RB_SWEEP_DELAY=8 ROWBLOCK_B200_LIB=variants/prof.so timeout 300 python tools/spmm_once.py 5 1 2 > gpurun_out/r02p/prof_d8.log 2>&1
RB_SWEEP_DELAY=8 ROWBLOCK_B200_LIB=variants/noload.so timeout 300 python tools/spmm_once.py 5 1 2 > gpurun_out/r02p/noload.log 2>&1
for d in 4 8; do (RB_SWEEP_DELAY=$d timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) > gpurun_out/r02s/bench5_d$d.json; done

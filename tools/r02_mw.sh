#!/bin/bash
mkdir -p gpurun_out/r02w
(timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or medium or two_streams" 2>&1 | tail -2) > gpurun_out/r02w/tests.log
ROWBLOCK_B200_LIB=variants/noload.so timeout 300 python tools/spmm_once.py 5 1 2 > gpurun_out/r02w/noload.log 2>&1
(timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) > gpurun_out/r02w/b5.json

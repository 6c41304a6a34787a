#!/bin/bash
mkdir -p gpurun_out/r02
./tools/l2bw/l2bw > gpurun_out/r02/l2bw2.txt 2>&1
(timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "medium or fullsize" 2>&1 | tail -25) > gpurun_out/r02/t2.log

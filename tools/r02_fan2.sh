#!/bin/bash
mkdir -p gpurun_out/fan
(timeout 600 python -m pytest tests/test_gpu_fanout.py -q 2>&1 | tail -30) > gpurun_out/fan/fanout_tests2.log
(timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -30) > gpurun_out/fan/gputests2.log
bash tools/r02_l2ab.sh 80

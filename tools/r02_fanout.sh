#!/bin/bash
# Fused all-gather (fan-out epilogue stores): GPU tests, whole GPU suite, config-5 bench (no regression).
mkdir -p gpurun_out/fan
(timeout 600 python -m pytest tests/test_gpu_fanout.py -x -q 2>&1 | tail -30) > gpurun_out/fan/fanout_tests.log
(timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30) > gpurun_out/fan/gputests.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 3 2> gpurun_out/fan/cfg5.err | tail -1 > gpurun_out/fan/cfg5.json

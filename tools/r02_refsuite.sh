#!/bin/bash
mkdir -p gpurun_out/r02r
(timeout 1800 python -m pytest tests/test_reference_suite.py tests/test_gpu_parity.py -x -q -s -k "reference or fp64" 2>&1 | tail -50) > gpurun_out/r02r/tests.log

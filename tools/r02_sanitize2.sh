#!/bin/bash
mkdir -p gpurun_out/r02z
(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config3.py -x -q -k "two_streams or nonfinite or split_hub or sweep or sparse or rmat" 2>&1 | tail -5) > gpurun_out/r02z/tests.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_cases.py > gpurun_out/r02z/racecheck.log 2>&1; echo "exit $?" >> gpurun_out/r02z/racecheck.log

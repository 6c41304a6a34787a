#!/bin/bash
# new GPU tests + compute-sanitizer passes over tools/sanitize_cases.py
mkdir -p gpurun_out/r02z
(timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "two_streams or nonfinite or split_hub or sweep" 2>&1 | tail -5) > gpurun_out/r02z/tests.log
timeout 300 python tools/sanitize_cases.py > gpurun_out/r02z/plain.log 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/r02z/$tool.log 2>&1
  echo "exit $?" >> gpurun_out/r02z/$tool.log
done

#!/bin/bash
mkdir -p gpurun_out/r02c
(timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_stats.py -x -q 2>&1 | tail -4) > gpurun_out/r02c/tests.log
for c in 1 2b 3; do
  (timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) > gpurun_out/r02c/b$c.json
  (RB_COMPACT_H=0 timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) > gpurun_out/r02c/b${c}_off.json
done

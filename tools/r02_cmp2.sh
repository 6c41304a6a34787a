#!/bin/bash
mkdir -p gpurun_out/r02c
for h in 2 4 8; do for c in 1 3; do
  (RB_COMPACT_H=$h timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) > gpurun_out/r02c/b${c}_h$h.json
done; done

#!/bin/bash
# Second L2 A/B: persisting set-aside at its B200 maximum (79 MB) with all / 55 % of B lines evict_last.
D=gpurun_out/l2ab2; mkdir -p $D
for i in 1 2; do
  for v in "RB_X=0" "RB_SWEEP_L2SET=79" "RB_SWEEP_L2SET=79 RB_SWEEP_BFRAC=55"; do
    tag=$(echo $v | tr ' =' '__')
    (env $v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) >> $D/$tag.json
  done
done

#!/bin/bash
# Random-row gather probe (ldg vs TMA bulk) and the gather-bound configs' bench lines with l2_gather.
mkdir -p gpurun_out/gp
timeout 300 ./tools/l2bw/gather_probe > gpurun_out/gp/gather_probe.txt 2>&1
for c in 3 2b 1; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 3 2> gpurun_out/gp/cfg$c.err | tail -1 > gpurun_out/gp/cfg$c.json
done

#!/bin/bash
# Quick GPU pass: tests, bench of the given configs, launch lists.  Usage: tools/gpu_check.sh "1 2b 3" "1 3"
CFGS=${1:-"1 2b 3"}; LL=${2:-""}
(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15) > gpurun_out/gputests.log
for c in $CFGS; do (timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) > gpurun_out/bench_cfg$c.log; done
for c in $LL; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:spmm --csv --log-file gpurun_out/ll_cfg$c.csv python tools/spmm_once.py $c > gpurun_out/once_cfg$c.log 2>&1; done

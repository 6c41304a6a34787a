#!/bin/bash
# sweep kernel: parity tests, config-5 bench (sweep on / off), ncu capture of the sweep kernel
mkdir -p gpurun_out/r02s
(timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or medium or shapes or shard" 2>&1 | tail -15) > gpurun_out/r02s/tests.log
(timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 5 2>&1 | tail -1) > gpurun_out/r02s/bench5.json
for d in 0 4 16; do (RB_SWEEP_DELAY=$d timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) > gpurun_out/r02s/bench5_d$d.json; done
(RB_SWEEP=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) > gpurun_out/r02s/bench5_off.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_sweep -s 2 -c 1 -o gpurun_out/r02s/ncu_sweep_cfg5 -f python tools/spmm_once.py 5 1 3 > gpurun_out/r02s/ncu.log 2>&1

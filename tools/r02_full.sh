#!/bin/bash
# full GPU suite + smoke + config-5 bench + ncu of the sweep kernel + launch list
mkdir -p gpurun_out/r02f
(timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5) > gpurun_out/r02f/gputests.log
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3) > gpurun_out/r02f/smoke.log
(timeout 900 python bench.py --steps 20 --warmup 5 --cpu-seconds 5 2>&1 | tail -1) > gpurun_out/r02f/bench5.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_sweep -s 2 -c 1 -o gpurun_out/r02f/ncu_sweep_cfg5 -f python tools/spmm_once.py 5 1 3 > gpurun_out/r02f/ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f/launches_cfg5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02f/ll.log 2>&1

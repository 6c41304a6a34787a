#!/bin/bash
mkdir -p gpurun_out/r02g
(timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3) > gpurun_out/r02g/gputests.log
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2) > gpurun_out/r02g/smoke.log
(timeout 900 python bench.py --steps 30 --warmup 5 --cpu-seconds 8 2>&1 | tail -1) > gpurun_out/r02g/cfg5.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_sweep -s 2 -c 1 -o gpurun_out/r02g/ncu_sweep64_cfg5 -f python tools/spmm_once.py 5 1 3 > gpurun_out/r02g/ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02g/launches_cfg5.csv python tools/spmm_once.py 5 1 3 > gpurun_out/r02g/ll.log 2>&1
timeout 900 python tools/shard_sim.py 5 2,4,8 10 2>&1 | tail -1 > gpurun_out/r02g/proj5.jsonl

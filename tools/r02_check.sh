#!/bin/bash
# Round-2 GPU pass: host facts, gpu tests, smoke, bench (config 5 default, both arms).
mkdir -p gpurun_out/r02
(free -g; nproc; grep "model name" /proc/cpuinfo | head -1; nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv) > gpurun_out/r02/host.txt 2>&1
(timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25) > gpurun_out/r02/gputests.log
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5) > gpurun_out/r02/smoke.log
(time timeout 900 python bench.py --steps 20 --warmup 5 2> gpurun_out/r02/bench5.err | tail -1) > gpurun_out/r02/bench5.json
(time timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 2> gpurun_out/r02/ref5.err | tail -1) > gpurun_out/r02/ref5.json

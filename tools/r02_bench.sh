#!/bin/bash
mkdir -p gpurun_out/r02
./tools/l2bw/l2bw > gpurun_out/r02/l2bw.txt 2>&1
( time timeout 900 python bench.py --steps 20 --warmup 5 2> gpurun_out/r02/bench5.err | tail -1 ) > gpurun_out/r02/bench5.json 2> gpurun_out/r02/bench5.time
( time timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 2> gpurun_out/r02/ref5.err | tail -1 ) > gpurun_out/r02/ref5.json 2> gpurun_out/r02/ref5.time

#!/bin/bash
# Round-end evidence: one bench line per config, the reference arm, a launch list and one full ncu
# capture of the config-5 short kernel.  Outputs land in gpurun_out/ (copied to profiles/ by hand).
mkdir -p gpurun_out/bench
for c in ${CFGS:-1 2 2b 3 4 5}; do
  timeout 900 python bench.py --config $c --steps 30 --warmup 3 --cpu-seconds 10 2> gpurun_out/bench/cfg$c.err | tail -1 > gpurun_out/bench/cfg$c.json
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 2> gpurun_out/bench/reference.err | tail -1 > gpurun_out/bench/reference_cfg2.json
if [ -n "$NCU5" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_short2 -s 3 -c 1 \
    -o gpurun_out/ncu_short2_cfg5 -f python tools/spmm_once.py 5 1 5 > gpurun_out/ncu5.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_cfg5.csv python tools/spmm_once.py 5 1 3 > gpurun_out/ll5.log 2>&1
fi

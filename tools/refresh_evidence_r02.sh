#!/bin/bash
# Round-2 evidence: one bench line per config, the reference arm (config 5), launch lists with DRAM
# bytes, and full ncu captures of each config's dominant kernel.  Outputs in gpurun_out/r02e/.
mkdir -p gpurun_out/r02e
for c in 5 1 2 2b 3 4; do
  extra=""; [ "$c" = "3" ] && extra="--no-cpu-baseline"
  timeout 900 python bench.py --config $c --steps 30 --warmup 5 --cpu-seconds 8 $extra 2> gpurun_out/r02e/cfg$c.err | tail -1 > gpurun_out/r02e/cfg$c.json
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 2> gpurun_out/r02e/reference.err | tail -1 > gpurun_out/r02e/reference_cfg5.json
for c in 2 4 5 3 2b 1; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02e/launches_cfg$c.csv python tools/spmm_once.py $c 1 3 > gpurun_out/r02e/ll$c.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_sweep -s 2 -c 1 -o gpurun_out/r02e/ncu_sweep_cfg5 -f python tools/spmm_once.py 5 1 3 > gpurun_out/r02e/ncu5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_csr -s 2 -c 1 -o gpurun_out/r02e/ncu_cmp_cfg3 -f python tools/spmm_once.py 3 1 3 > gpurun_out/r02e/ncu3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_tall2 -s 2 -c 1 -o gpurun_out/r02e/ncu_tall2_cfg2 -f python tools/spmm_once.py 2 1 3 > gpurun_out/r02e/ncu2.log 2>&1

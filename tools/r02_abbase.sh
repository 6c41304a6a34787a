#!/bin/bash
# Same-box A/B of config 5: the round-2 closing build (variants/base = commit 0d133c1) against the
# current tree (fan-out epilogues + L2 knobs).  Bench lines + one ncu metric pass of the sweep kernel each.
D=gpurun_out/abbase; mkdir -p $D
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_sector_hit_rate.pct
for i in 1 2 3; do
  (cd variants/base && timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) >> $D/base.json
  (timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) >> $D/cur.json
done
(cd variants/base && timeout 600 ncu --metrics $M --clock-control none -k regex:spmm_sweep -c 3 --csv python ../../tools/spmm_once.py 5 1 3) > $D/ncu_base.csv 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:spmm_sweep -c 3 --csv python tools/spmm_once.py 5 1 3 > $D/ncu_cur.csv 2>&1

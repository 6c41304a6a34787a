#!/bin/bash
# (1) config 5 same-box A/B: closing build (variants/base) vs current; ncu metrics of the sweep kernel.
# (2) CSR engine: per-item (RB_CSR_PF=0) vs cross-item prefetch (default) vs prefetch at 3 CTAs/SM
#     (variants/pf3) on configs 3 / 2b / 1.  (3) parity tests of the compact / CSR paths.
D=gpurun_out/ab2; mkdir -p $D
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_sector_hit_rate.pct
for i in 1 2; do
  (cd variants/base && timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) >> $D/c5_base.json
  (timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) >> $D/c5_cur.json
done
timeout 600 ncu --metrics $M --clock-control none -k regex:spmm_sweep -c 2 --csv python tools/spmm_once.py 5 1 2 > $D/ncu5_cur.csv 2>&1
for c in 3 2b 1; do
  for i in 1 2; do
    (RB_CSR_PF=0 timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) >> $D/c${c}_pf0.json
    (timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) >> $D/c${c}_pf1.json
    (ROWBLOCK_B200_LIB=$PWD/variants/pf3/paper_2202_05868_b200/librowblock_b200.so timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) >> $D/c${c}_pf3.json
  done
done
(timeout 1200 python -m pytest tests/test_gpu_config3.py tests/test_gpu_parity.py tests/test_gpu_fanout.py -q -x 2>&1 | tail -5) > $D/tests.log

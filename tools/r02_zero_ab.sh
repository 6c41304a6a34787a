#!/bin/bash
# Batched zero_rows_kernel: parity (the GPU suite's parity + full-size files) and a same-box config-3
# A/B against the previous build (variants/base), plus the new kernel's launch times under ncu.
D=gpurun_out/r02zr; mkdir -p $D; rm -f $D/*.json
(timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fanout.py -m gpu -q -x 2>&1 | tail -4) > $D/tests.log
for i in 1 2 3; do
  (cd variants/base && timeout 300 python bench.py --config 3 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | tail -1) >> $D/c3_base.json
  (timeout 300 python bench.py --config 3 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | tail -1) >> $D/c3_new.json
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:zero_rows --log-file $D/launches_zero_cfg3.csv python tools/spmm_once.py 3 1 3 > $D/ll3.log 2>&1

#!/bin/bash
# CSR engine: runtime-chunk instance for 32-lane groups (configs 2b, 1), single-claim instance for
# 16-lane groups (config 3), against variants/base.  Parity first, then same-box alternating runs.
D=gpurun_out/r02ch4; mkdir -p $D; rm -f $D/*.json
(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -3) > $D/tests.log
run() { timeout 300 python bench.py --config $1 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | tail -1; }
for c in 2b 1 3; do for i in 1 2 3; do
  (cd variants/base && run $c) >> $D/c${c}_base.json
  run $c >> $D/c${c}_new.json
done; done

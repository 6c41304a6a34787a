#!/bin/bash
# CSR engine with runtime claim chunks (csr_claim_chunk: 2 for uniform, long work lists, else 1)
# against variants/base (one item per claim): parity, then same-box alternating configs 2b, 3, 1.
D=gpurun_out/r02ch3; mkdir -p $D; rm -f $D/*.json
(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -3) > $D/tests.log
run() { timeout 300 python bench.py --config $1 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | tail -1; }
for c in 2b 3 1; do for i in 1 2; do
  (cd variants/base && run $c) >> $D/c${c}_base.json
  run $c >> $D/c${c}_new.json
done; done

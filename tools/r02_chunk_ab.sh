#!/bin/bash
# CSR engine: items claimed RB_CSR_CHUNK at a time (4 = current tree, 2 = variants/ch2, 1 = variants/base).
# Parity of the CSR / compact paths, then same-box alternating bench lines for configs 3, 2b, 1.
D=gpurun_out/r02ch; mkdir -p $D; rm -f $D/*.json
(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -3) > $D/tests.log
run() { timeout 300 python bench.py --config $1 --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | tail -1; }
for c in 3 2b 1; do for i in 1 2; do
  (cd variants/base && run $c) >> $D/c${c}_base.json
  (cd variants/ch2 && run $c) >> $D/c${c}_ch2.json
  run $c >> $D/c${c}_ch4.json
done; done

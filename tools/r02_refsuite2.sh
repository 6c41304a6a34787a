#!/bin/bash
# The reference's own hot-path test files against the drop-in (needs baseline/_ref from
# tools/install_reference.sh), plus repeat config-5 bench lines for box-to-box spread.
D=gpurun_out/r02y; mkdir -p $D
(timeout 1500 python -m pytest tests/test_reference_suite.py -m gpu -q -rs 2>&1 | tail -15) > $D/refsuite.log
for i in 1 2; do timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 10 2> $D/cfg5_$i.err | tail -1 > $D/cfg5_$i.json; done

#!/bin/bash
# Final verification of the build of record: whole GPU suite (reference suite included, baseline/_ref
# shipped), smoke, default bench line (config 5) and config 3.  Outputs in gpurun_out/r02v2/.
D=gpurun_out/r02v2; mkdir -p $D
(timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4) > $D/gputests.log
(timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2) > $D/smoke.log
timeout 900 python bench.py 2> $D/default.err | tail -1 > $D/default.json
timeout 900 python bench.py --config 3 --steps 30 --warmup 5 --no-cpu-baseline 2> $D/cfg3.err | tail -1 > $D/cfg3.json
timeout 900 python bench.py --config 2b --steps 30 --warmup 5 --cpu-seconds 8 2> $D/cfg2b.err | tail -1 > $D/cfg2b.json

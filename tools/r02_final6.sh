#!/bin/bash
# Round-2 closing run: GPU tests, smoke, then every bench line, launch list and ncu capture.
mkdir -p gpurun_out/r02e
(timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3) > gpurun_out/r02e/gputests.log
(timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2) > gpurun_out/r02e/smoke.log
./tools/refresh_evidence_r02.sh

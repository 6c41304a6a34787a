#!/bin/bash
# Round-2 closing run after the fused-gather change: GPU tests, smoke, every bench line, reference
# arm, launch lists and ncu captures (tools/refresh_evidence_r02.sh -> gpurun_out/r02e/).
mkdir -p gpurun_out/r02e
(timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3) > gpurun_out/r02e/gputests.log
(timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2) > gpurun_out/r02e/smoke.log
./tools/refresh_evidence_r02.sh

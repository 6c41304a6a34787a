#!/bin/bash
# Closing evidence of round 2 (re-entry session): GPU tests, smoke, every config's bench line, the
# reference arm, launch lists with DRAM bytes, and full ncu captures of the config-5 sweep and
# config-3 CSR kernels.  Outputs in gpurun_out/r02z/.
D=gpurun_out/r02z; mkdir -p $D
(timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -15) > $D/gputests.log
(timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2) > $D/smoke.log
for c in 5 1 2 2b 3 4; do
  extra=""; [ "$c" = "3" ] && extra="--no-cpu-baseline"
  timeout 900 python bench.py --config $c --steps 30 --warmup 5 --cpu-seconds 8 $extra 2> $D/cfg$c.err | tail -1 > $D/cfg$c.json
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 2> $D/reference.err | tail -1 > $D/reference_cfg5.json
for c in 5 3 2; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $D/launches_cfg$c.csv python tools/spmm_once.py $c 1 3 > $D/ll$c.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_sweep -s 2 -c 1 -o $D/ncu_sweep_cfg5 -f python tools/spmm_once.py 5 1 3 > $D/ncu5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_csr -s 2 -c 1 -o $D/ncu_cmp_cfg3 -f python tools/spmm_once.py 3 1 3 > $D/ncu3.log 2>&1

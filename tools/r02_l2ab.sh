#!/bin/bash
# Config-5 sweep kernel L2 policy A/B: B lines evict_last share (RB_SWEEP_BFRAC), persisting-L2
# set-aside (RB_SWEEP_L2SET, MB), C stores evict_first (RB_SWEEP_CST).  Lines in gpurun_out/l2ab/.
D=gpurun_out/l2ab; mkdir -p $D
python - > $D/l2props.txt 2>&1 <<'PY'
import ctypes
rt = ctypes.CDLL("libcudart.so.12") if True else None
v = ctypes.c_int(0)
for name, attr in (("l2_bytes", 89), ("max_persisting_l2_bytes", 108), ("max_access_policy_window", 109)):
    rc = rt.cudaDeviceGetAttribute(ctypes.byref(v), attr, 0)
    print(name, v.value, "rc", rc)
PY
MAXMB=${1:-80}
for i in 1 2; do
  for v in "RB_X=0" "RB_SWEEP_CST=1" "RB_SWEEP_L2SET=$MAXMB" "RB_SWEEP_L2SET=$MAXMB RB_SWEEP_BFRAC=50" "RB_SWEEP_BFRAC=50" "RB_SWEEP_L2SET=$MAXMB RB_SWEEP_BFRAC=35"; do
    tag=$(echo $v | tr ' =' '__')
    (env $v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) >> $D/$tag.json
  done
done

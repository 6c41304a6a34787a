#!/bin/bash
# A/B of an env setting on one config's bench: tools/ab.sh "ENV=a" "ENV=b" [reps] [config] [tag]
# Lines append to gpurun_out/ab/<tag>/<setting>.json (the tag directory is cleared first).
R=${3:-3}; C=${4:-5}; T=${5:-c$C}
D=gpurun_out/ab/$T; mkdir -p $D; rm -f $D/*.json
for i in $(seq $R); do for v in "$1" "$2"; do
  (env $v timeout 300 python bench.py --config $C --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) >> $D/"$(echo $v | tr '=/.' '___')".json
done; done

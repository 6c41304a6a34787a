#!/bin/bash
# A/B of an env knob on the config-5 bench: tools/ab.sh "ENV=a" "ENV=b" [reps] [config]
mkdir -p gpurun_out/ab; rm -f gpurun_out/ab/*.json
R=${3:-3}; C=${4:-5}
for i in $(seq $R); do for v in "$1" "$2"; do
  (env $v timeout 300 python bench.py --config $C --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1) >> gpurun_out/ab/"$(echo $v | tr '=/.' '___')".json
done; done

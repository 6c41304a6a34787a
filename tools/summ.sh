#!/bin/bash
# Summarise tools/gpu_check.sh outputs
tail -3 gpurun_out/gputests.log
for f in gpurun_out/bench_cfg*.log; do python - $f <<'PY'
import json,sys
t=open(sys.argv[1]).read().strip().splitlines()
try: d=json.loads(t[-1])
except Exception: print(sys.argv[1], t[-3:]); sys.exit()
print(sys.argv[1], d['value'], 'ms', d['ms_per_step'], 'e2e',d['e2e']['value'], 'launches', d['gpu_launches'], 'frac', d['roofline']['frac'])
PY
done
for f in gpurun_out/ll_cfg*.csv; do python - $f <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:]:
    if not r[vi].replace(',','').replace('.','').isdigit(): continue
    print(sys.argv[1], r[ki][:80], r[vi])
PY
done

"""Time the SpMM of one config under environment variants (plan knobs read at plan creation).

python tools/short_probe.py cfg5 "RB_SHORT_CACHE=100" "RB_SHORT_CACHE=101 RB_SHORT_NS=128" ...
Each variant: fresh plan, 3 warm-up executes, median of 10 CUDA-event timed executes.
"""
import os, sys, torch
sys.path.insert(0, '.')
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import block_1sa_device, DeviceVbr
from paper_2202_05868_b200.types import MergePolicy

name = sys.argv[1]
dA, bounds, cfg, meta = synth.make(name, scale=1, device="cuda")
dg = block_1sa_device(dA, bounds, MergePolicy(tau=cfg.tau), True)
B = synth.make_b(cfg, dA.n_cols, cfg.precision, device="cuda")
dv = DeviceVbr.build(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=(cfg.precision,))
out = torch.empty((dA.n_rows, cfg.N), dtype=torch.float32, device="cuda")
ref = None
for var in sys.argv[2:]:
    keys = []
    for kv in var.split():
        k, v = kv.split("=")
        os.environ[k] = v
        keys.append(k)
    DeviceVbr._destroy_plans(dv._plans)
    for _ in range(3):
        dv.spmm(B, out=out, precision=cfg.precision)
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); dv.spmm(B, out=out, precision=cfg.precision); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort()
    if ref is None:
        ref = out.clone()
    err = float(((out - ref).abs() / ref.abs().clamp_min(1e-3)).max())
    bad = int(((out - ref).abs() > 1e-4 * ref.abs().clamp_min(1e-3)).sum())
    print(f"{name} [{var}] median {ts[5]:.3f} ms  min {ts[0]:.3f}  max_rel_vs_first {err:.2e} n_bad {bad}", flush=True)
    for k in keys:
        del os.environ[k]

"""Build config <name> at <scale> and run its SpMM <reps> times (for ncu launch lists)."""
import os, sys, torch
sys.path.insert(0, '.')
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import block_1sa_device, DeviceVbr
from paper_2202_05868_b200.types import MergePolicy
name = sys.argv[1]; scale = int(sys.argv[2]) if len(sys.argv) > 2 else 1; reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
tau = float(sys.argv[4]) if len(sys.argv) > 4 else None
dA, bounds, cfg, meta = synth.make(name, scale=scale, device="cuda")
dg = block_1sa_device(dA, bounds, MergePolicy(tau=tau if tau is not None else cfg.tau), True)
B = synth.make_b(cfg, dA.n_cols, cfg.precision, device="cuda")
dv = DeviceVbr.build(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=(cfg.precision,))
print(dv.plan_info(cfg.N, cfg.precision))
rp, bp, bc = dv.host_structure()
import numpy as np
h = np.diff(rp); nb = np.diff(bp)
for lo, hi in [(1, 1), (2, 2), (3, 4), (5, 8), (9, 16), (17, 128), (129, 1 << 30)]:
    m = (h >= lo) & (h <= hi)
    print(f"h in [{lo},{hi}]: rows {h[m].sum()} block rows {m.sum()} blocks {nb[m].sum()}")
torch.cuda.synchronize()
for _ in range(reps): C = dv.spmm(B, precision=cfg.precision)
torch.cuda.synchronize()

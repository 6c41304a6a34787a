import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import block_1sa_device, DeviceVbr
from paper_2202_05868_b200.types import MergePolicy
dA, bounds, cfg, meta = synth.make("3", scale=1, device="cuda")
dg = block_1sa_device(dA, bounds, MergePolicy(tau=cfg.tau), True)
dv = DeviceVbr.build(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=(cfg.precision,))
perm = dv.row_perm64.cpu().numpy()
rnnz = np.diff(dA.row_ptr.cpu().numpy())
W = 8
los = [dv.plan_info(cfg.N, cfg.precision, k, W)["row_begin_perm"] for k in range(W)] + [dA.n_rows]
rp, bp, bc = dv.host_structure()
for k in range(W):
    lo, hi = los[k], los[k + 1]
    rows = perm[lo:hi]
    g0 = np.searchsorted(rp, lo, 'right') - 1; g1 = np.searchsorted(rp, hi, 'left')
    print(k, lo, hi, "nnz", int(rnnz[rows].sum()), "blocks", int(bp[g1] - bp[g0]), "max_row_nnz", int(rnnz[rows].max()) if len(rows) else 0)

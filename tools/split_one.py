import os, sys, torch
sys.path.insert(0, '.')
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import block_1sa_device, DeviceVbr
from paper_2202_05868_b200.types import MergePolicy
dA, bounds, cfg, meta = synth.make(sys.argv[1], scale=1, device="cuda")
dg = block_1sa_device(dA, bounds, MergePolicy(tau=cfg.tau), True)
B = synth.make_b(cfg, dA.n_cols, "bf16", device="cuda")
dv = DeviceVbr.build(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=("bf16",))
for _ in range(3): C = dv.spmm(B)
torch.cuda.synchronize()

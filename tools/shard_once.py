import sys, torch
sys.path.insert(0, '.')
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import block_1sa_device, DeviceVbr
from paper_2202_05868_b200.types import MergePolicy
dA, bounds, cfg, meta = synth.make("3", scale=1, device="cuda")
dg = block_1sa_device(dA, bounds, MergePolicy(tau=cfg.tau), True)
dv = DeviceVbr.build(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=(cfg.precision,))
B = synth.make_b(cfg, dA.n_cols, cfg.precision, device="cuda")
C = torch.empty((dA.n_rows, cfg.N), dtype=torch.float32, device="cuda")
for k in [0, 1, 4]:
    for _ in range(2): dv.spmm(B, out=C, precision=cfg.precision, shard=k, n_shards=8)
    torch.cuda.synchronize()
    print("shard", k, dv.plan_info(cfg.N, cfg.precision, k, 8), flush=True)

"""Time one shard's plan of a config under environment variants: python tools/shard_probe.py cfg k W "ENV=..." ..."""
import os, sys, torch
sys.path.insert(0, '.')
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import block_1sa_device, DeviceVbr
from paper_2202_05868_b200.types import MergePolicy
name, k, W = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
dA, bounds, cfg, meta = synth.make(name, scale=1, device="cuda")
dg = block_1sa_device(dA, bounds, MergePolicy(tau=cfg.tau), True)
dv = DeviceVbr.build(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=(cfg.precision,))
B = synth.make_b(cfg, dA.n_cols, cfg.precision, device="cuda")
C = torch.empty((dA.n_rows, cfg.N), dtype=torch.float32, device="cuda")
for var in sys.argv[4:]:
    keys = []
    for kv in var.split():
        a, b = kv.split("=")
        os.environ[a] = b
        keys.append(a)
    DeviceVbr._destroy_plans(dv._plans)
    for _ in range(3): dv.spmm(B, out=C, precision=cfg.precision, shard=k, n_shards=W)
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); dv.spmm(B, out=C, precision=cfg.precision, shard=k, n_shards=W); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(name, k, W, var, "median %.3f ms" % sorted(ts)[5], flush=True)
    for a in keys: del os.environ[a]

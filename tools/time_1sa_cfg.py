"""Time the device 1-SA (and VBR build) of a config at full size: python tools/time_1sa_cfg.py <cfg> [tau,...]"""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import block_1sa_device, DeviceVbr
from paper_2202_05868_b200.types import MergePolicy
dA, bounds, cfg, meta = synth.make(sys.argv[1], scale=1, device="cuda")
taus = [float(t) for t in sys.argv[2].split(",")] if len(sys.argv) > 2 else [cfg.tau]
block_1sa_device(dA, bounds, MergePolicy(tau=taus[0]), True)  # warm (module load, allocations)
torch.cuda.synchronize()
for tau in taus:
    t0 = time.perf_counter()
    dg = block_1sa_device(dA, bounds, MergePolicy(tau=tau), True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    dv = DeviceVbr.build(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=(cfg.precision,))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"cfg {sys.argv[1]} tau={tau} H={dg.n_groups} 1sa={t1 - t0:.4f}s vbr={t2 - t1:.4f}s", flush=True)

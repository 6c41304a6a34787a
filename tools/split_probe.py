"""Probe the tall-kernel split-K tail: time config 2/4 at RB_TALL_SPLIT=1..4 and compare C."""
import os, sys, time, torch
sys.path.insert(0, '.')
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import block_1sa_device, DeviceVbr
from paper_2202_05868_b200.types import MergePolicy
cfgname = sys.argv[1]
dA, bounds, cfg, meta = synth.make(cfgname, scale=1, device="cuda")
dg = block_1sa_device(dA, bounds, MergePolicy(tau=cfg.tau), True)
B = synth.make_b(cfg, dA.n_cols, "bf16", device="cuda")
ref = None
for s in sys.argv[2].split(','):
    os.environ["RB_TALL_SPLIT"] = s
    dv = DeviceVbr.build(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=("bf16",))
    info = dv.plan_info(cfg.N, "bf16")
    C = dv.spmm(B); torch.cuda.synchronize()
    st = torch.cuda.Event(enable_timing=True); en = torch.cuda.Event(enable_timing=True)
    st.record()
    for _ in range(10): dv.spmm(B, out=C)
    en.record(); torch.cuda.synchronize()
    ms = st.elapsed_time(en) / 10
    if ref is None: ref = C.clone()
    d = (C - ref).abs().max().item()
    print(f"split={s} units={info['n_items_tall']} ms={ms:.4f} maxdiff_vs_first={d:.3e}", flush=True)

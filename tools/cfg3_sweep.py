"""Config 3 (R-MAT 2^20/scale, Δ=32, N=128) τ sweep on the device: 1-SA, VBR build and SpMM times.

    python tools/cfg3_sweep.py <scale> <tau,tau,...>
"""
import time, torch, sys
sys.path.insert(0, '.')
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import block_1sa_device, DeviceVbr
from paper_2202_05868_b200.types import MergePolicy
dA, bounds, cfg, meta = synth.make("3", scale=int(sys.argv[1]), device="cuda")
print("n", dA.n_rows, "nnz", dA.nnz, flush=True)
for tau in [float(x) for x in sys.argv[2].split(",")]:
    torch.cuda.synchronize(); t = time.time()
    dg = block_1sa_device(dA, bounds, MergePolicy(tau=tau), True)
    torch.cuda.synchronize(); t1 = time.time()
    dv = DeviceVbr.build(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=("bf16",))
    torch.cuda.synchronize(); t2 = time.time()
    B = synth.make_b(cfg, dA.n_cols, "bf16", device="cuda")
    C = dv.spmm(B); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): dv.spmm(B, out=C)
    e.record(); torch.cuda.synchronize(); ms = s.elapsed_time(e) / 5
    print(f"tau={tau} H={dg.n_groups} 1sa={t1-t:.2f}s vbr={t2-t1:.2f}s blocks={dv.n_blocks} spmm={ms:.3f}ms eff={2*dA.nnz*128/ms/1e9:.1f}TF/s area={dv.stored_area()}", flush=True)

"""Repeat the bench's e2e pipeline measurement (config 2) several times in one process."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import block_1sa_device, DeviceVbr
from paper_2202_05868_b200.multiply import SpmmPipeline, pinned_dense
from paper_2202_05868_b200.types import MergePolicy
dA, bounds, cfg, meta = synth.make("2", scale=1, device="cuda")
dg = block_1sa_device(dA, bounds, MergePolicy(tau=cfg.tau), True)
dv = DeviceVbr.build(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=("bf16",))
B = synth.make_b(cfg, dA.n_cols, "bf16", device="cuda")
N = B.shape[1]
Bh = [B.double().cpu().pin_memory() for _ in range(2)]
Ch = [pinned_dense(dA.n_rows, N) for _ in range(2)]
pipe = SpmmPipeline(dv, N, "bf16")
for steps in [int(x) for x in sys.argv[1].split(',')]:
    for k in range(2): pipe.step(k, Bh[k % 2], Ch[k % 2])
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record(pipe.s_in)
    for k in range(steps): pipe.step(k, Bh[k % 2], Ch[k % 2])
    t1 = time.perf_counter()
    e.record(pipe.s_out)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"steps={steps} ms/step={s.elapsed_time(e)/steps:.3f} enqueue={1e3*(t1-t0)/steps:.3f}ms wall={1e3*(t2-t0)/steps:.3f}", flush=True)

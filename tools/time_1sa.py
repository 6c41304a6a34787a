"""Time device block_1sa on a synthetic config: python tools/time_1sa.py <config> <scale> <tau>"""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import block_1sa_device
from paper_2202_05868_b200.types import MergePolicy
dA, bounds, cfg, meta = synth.make(sys.argv[1], scale=int(sys.argv[2]), device="cuda")
tau = float(sys.argv[3])
for rep in range(2):
    torch.cuda.synchronize(); t = time.time()
    dg = block_1sa_device(dA, bounds, MergePolicy(tau=tau), True)
    torch.cuda.synchronize()
    print(f"cfg{sys.argv[1]} n={dA.n_rows} tau={tau} H={dg.n_groups} t={time.time()-t:.3f}s", flush=True)

"""Config <name>: run the GPU spmm_csr comparator <reps> times (ncu target)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2202_05868_b200 import synth
dA, bounds, cfg, meta = synth.make(sys.argv[1], scale=1, device="cuda")
B = synth.make_b(cfg, dA.n_cols, cfg.precision, device="cuda")
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    C = dA.spmm(B, precision=cfg.precision)
torch.cuda.synchronize()

import os, sys, threading
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
os.environ["RB_TALL_SPLIT"] = "2"
import numpy as np, torch
import paper_2202_05868_b200 as rb
from conftest import load_golden
c = load_golden("cfg4_s8")
A = rb.CsrMatrix(int(c["n_rows"]), int(c["n_cols"]), c["row_ptr"], c["col_idx"], c["values"])
q = rb.ColumnPartition(int(c["n_cols"]), c["boundaries"])
V = rb.vbr_from_grouping(A, rb.block_1sa(A, q, rb.MergePolicy(tau=0.7), True), q)
dv = V.device
print(dv.plan_info(512, "bf16"))
g = torch.Generator(device="cuda").manual_seed(5)
Bs = [torch.rand((A.n_cols, 512), device="cuda", generator=g).to(torch.bfloat16) for _ in range(4)]
refs = [dv.spmm(B, precision="bf16").clone() for B in Bs]
torch.cuda.synchronize()
for rep in range(3):
    again = [dv.spmm(B, precision="bf16").clone() for B in Bs]
    torch.cuda.synchronize()
    print("same-stream rerun equal:", [torch.equal(a, b) for a, b in zip(again, refs)])
streams = [torch.cuda.Stream() for _ in range(2)]
outs = [torch.empty_like(r) for r in refs]
def worker(k):
    st = streams[k % 2]
    with torch.cuda.stream(st):
        for _ in range(4):
            dv.spmm(Bs[k], out=outs[k], precision="bf16", stream=st)
    st.synchronize()
for trial in range(3):
    ths = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    [t.start() for t in ths]; [t.join() for t in ths]
    torch.cuda.synchronize()
    print("threads:", [(torch.equal(outs[k], refs[k]), (outs[k] - refs[k]).abs().max().item()) for k in range(4)])

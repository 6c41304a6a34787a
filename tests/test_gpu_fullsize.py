"""Full-size (BASELINE.json configs) GPU checks through size-independent properties.

At the bench sizes the CPU oracle cannot produce C in test time, so C is checked by a
checksum of checksums: for random vectors r, C·r must equal A·(B·r) computed in float64 on the
device (torch sparse CSR), within the bf16-input/fp32-accumulate bound
|C·r - A(B·r)| <= 1e-3 · (|A|·|B|)·|r|  (inputs are pre-rounded to bf16, so only fp32
accumulation error remains).  Rows of empty block rows must be exactly 0.  The 1-SA structure of
config 2/4/5 is checked against the C oracle (bit-exact)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import DeviceVbr, block_1sa_device
from paper_2202_05868_b200.types import MergePolicy

pytestmark = pytest.mark.gpu


def _check_product(dA, dv, B, C, n_vec=3):
    rp = dA.row_ptr
    A = torch.sparse_csr_tensor(rp, dA.col_idx, dA.values, size=(dA.n_rows, dA.n_cols))
    Aabs = torch.sparse_csr_tensor(rp, dA.col_idx, dA.values.abs(), size=(dA.n_rows, dA.n_cols))
    B64 = B.double()
    g = torch.Generator(device="cuda").manual_seed(3)
    for _ in range(n_vec):
        r = torch.randn(B.shape[1], 1, device="cuda", dtype=torch.float64, generator=g)
        lhs = C.double() @ r
        rhs = A @ (B64 @ r)
        bound = Aabs @ (B64.abs() @ r.abs())
        assert torch.all((lhs - rhs).abs() <= 1e-3 * bound + 1e-12), float(((lhs - rhs).abs() / (bound + 1e-12)).max())


@pytest.mark.parametrize("name,scale", [("2", 1), ("4", 1), ("5", 4), ("2b", 4), ("1", 1)])
def test_fullsize_structure_and_product(name, scale):
    dA, bounds, cfg, meta = synth.make(name, scale=scale, device="cuda")
    dg = block_1sa_device(dA, bounds, MergePolicy(tau=cfg.tau), True)
    if dA.n_rows <= 40000:
        ref = oracle.block_1sa_arrays(dA.row_ptr.cpu().numpy(), dA.col_idx.cpu().numpy(), bounds, tau=cfg.tau)
        assert ref["n_groups"] == dg.n_groups
        assert np.array_equal(ref["row_perm"], dg.row_perm.cpu().numpy())
        assert np.array_equal(ref["group_ptr"], dg.group_ptr[: dg.n_groups + 1].cpu().numpy())
    dv = DeviceVbr.build(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=(cfg.precision,))
    B = synth.make_b(cfg, dA.n_cols, cfg.precision, device="cuda")
    C = dv.spmm(B, precision=cfg.precision)
    C2 = dv.spmm(B, precision=cfg.precision)
    torch.cuda.synchronize()
    assert torch.equal(C, C2)  # deterministic
    _check_product(dA, dv, B, C)
    empty = (dA.row_ptr[1:] - dA.row_ptr[:-1]) == 0
    assert torch.all(C[empty] == 0)

"""Config 3 (R-MAT, Δ=32, τ sweep): the sparse 1-SA path vs the pruned C oracle (bit-exact).

The pruned oracle (oracle/rowblock_oracle.c: orc_block_1sa_pruned) is itself pinned against the
reference on every golden case (tests/test_oracle.py::test_pruned_oracle_matches_golden)."""
import numpy as np
import pytest

import oracle
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import block_1sa_device
from paper_2202_05868_b200.types import MergePolicy

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale,tau", [(64, 0.3), (64, 0.9), (16, 0.3), (16, 0.5), (16, 0.9)])
def test_rmat_block_1sa_matches_pruned_oracle(scale, tau):
    dA, bounds, cfg, meta = synth.make("3", scale=scale, device="cuda")
    dg = block_1sa_device(dA, bounds, MergePolicy(tau=tau), True)
    ref = oracle.block_1sa_arrays(dA.row_ptr.cpu().numpy(), dA.col_idx.cpu().numpy(), bounds, tau=tau, pruned=True)
    assert dg.n_groups == ref["n_groups"]
    assert np.array_equal(dg.row_perm.cpu().numpy(), ref["row_perm"])
    assert np.array_equal(dg.group_ptr[: dg.n_groups + 1].cpu().numpy(), ref["group_ptr"])
    assert np.array_equal(dg.seed_size[: dg.n_groups].cpu().numpy(), ref["seed_size"])
    pp = dg.pattern_ptr[: dg.n_groups + 1].cpu().numpy()
    assert np.array_equal(pp, ref["pattern_ptr"])
    assert np.array_equal(dg.pattern_idx[: pp[-1]].cpu().numpy(), ref["pattern_idx"])

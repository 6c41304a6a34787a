"""Pin the CPU oracle (oracle/, test infrastructure) against reference-generated golden vectors.

The fixtures in tests/golden/ were produced by running the reference rowblock
v0.1.0 itself (tests/golden/make_golden.py).  If these pass, the oracle is a
faithful restatement of block_1sa (blocking.py:283-306), vbr_from_grouping's
block structure (vbr.py:88-125) and spmm_vbr (multiply.py:72-97).
"""
import numpy as np
import pytest

import oracle
from conftest import MEDIUM, golden_b, load_golden


def _check_structure(case):
    out = oracle.block_1sa_arrays(case["row_ptr"], case["col_idx"], case["boundaries"], tau=float(case["tau"]),
                                  similarity="cosine" if int(case["cosine"]) else "jaccard",
                                  bounded=bool(case["bounded"]), pattern_update=bool(case["pattern_update"]),
                                  use_compression=bool(case["use_compression"]))
    assert np.array_equal(out["group_of"], case["group_of"])
    assert np.array_equal(out["row_perm"], case["row_perm"])
    assert np.array_equal(out["group_ptr"], case["row_partition"])
    assert np.array_equal(out["seed_size"], case["seed_size"])
    assert np.array_equal(out["pattern_ptr"], case["pattern_ptr"])
    assert np.array_equal(out["pattern_idx"], case["pattern_idx"])
    bp, bc = oracle.vbr_blocks(case["row_ptr"], case["col_idx"], case["boundaries"], case["row_perm"],
                               case["row_partition"])
    assert np.array_equal(bp, case["blk_ptr"])
    assert np.array_equal(bc, case["blk_col"])
    return out


def test_oracle_structure_small(golden_small):
    assert len(golden_small) > 140
    for name, case in golden_small.items():
        try:
            _check_structure(case)
        except AssertionError as e:  # pragma: no cover - diagnostic
            raise AssertionError(f"case {name}") from e


def test_oracle_spmm_small(golden_small):
    for name, case in golden_small.items():
        B = golden_b(case)
        if B is None or "C" not in case:
            continue
        pay = oracle.vbr_payloads(case["row_ptr"], case["col_idx"], case["values"], case["boundaries"],
                                  case["row_perm"], case["row_partition"], case["blk_ptr"], case["blk_col"])
        C = oracle.spmm_vbr_np(pay, case["row_perm"], case["row_partition"], case["boundaries"], B)
        C8 = oracle.spmm_vbr_np(pay, case["row_perm"], case["row_partition"], case["boundaries"], B, threads=8)
        assert np.array_equal(C, C8), name
        ref = case["C"]
        nz = ref != 0
        assert np.all(np.abs(C - ref)[nz] <= 1e-12 * np.abs(ref)[nz]), name
        assert np.array_equal(C[~nz], ref[~nz]), name


@pytest.mark.parametrize("name", MEDIUM)
def test_oracle_structure_medium(name):
    case = load_golden(name)
    _check_structure(case)
    B = golden_b(case)
    if B is not None:
        pay = oracle.vbr_payloads(case["row_ptr"], case["col_idx"], case["values"], case["boundaries"],
                                  case["row_perm"], case["row_partition"], case["blk_ptr"], case["blk_col"])
        C = oracle.spmm_vbr_np(pay, case["row_perm"], case["row_partition"], case["boundaries"], B, threads=4)
        r = np.random.default_rng(7).standard_normal(B.shape[1])
        np.testing.assert_allclose(C @ r, case["C_dot_r"], rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(C.sum(axis=1), case["C_rowsum"], rtol=1e-12, atol=1e-12)


def test_pruned_oracle_matches_golden(golden_small):
    """orc_block_1sa_pruned (the config-3-scale oracle) == the reference on every golden case."""
    from conftest import load_golden
    cases = list(golden_small.items()) + [(m, load_golden(m)) for m in MEDIUM]
    for name, c in cases:
        a = oracle.block_1sa_arrays(c["row_ptr"], c["col_idx"], c["boundaries"], tau=float(c["tau"]),
                                    similarity="cosine" if int(c["cosine"]) else "jaccard",
                                    bounded=bool(c["bounded"]), pattern_update=bool(c["pattern_update"]),
                                    use_compression=bool(c["use_compression"]), pruned=True)
        assert np.array_equal(a["row_perm"], c["row_perm"]), name
        assert np.array_equal(a["group_ptr"], c["row_partition"]), name
        assert np.array_equal(a["seed_size"], c["seed_size"]), name
        assert np.array_equal(a["pattern_ptr"], c["pattern_ptr"]), name
        assert np.array_equal(a["pattern_idx"], c["pattern_idx"]), name

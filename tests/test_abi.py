"""C-ABI checks that need no GPU: the library loads, exports every symbol include/rowblock_b200.h
declares, validates arguments before touching the device, and the host shard planner is sound."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2202_05868_b200 import _lib as L
from paper_2202_05868_b200 import dist as rbdist
from conftest import ROOT, load_golden


def header_symbols():
    src = open(os.path.join(ROOT, "include", "rowblock_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), f"missing export {s}"
    assert lib.rb_abi_version() == 1


def test_policy_validation_before_device_work():
    lib = L.lib()
    H = ctypes.c_int64(0)
    rc = lib.rb_block_1sa(4, 4, 0, None, None, None, 1, 1.5, L.RB_JACCARD, 1, 1, 1, None, 0, None, None, None,
                          None, None, None, ctypes.byref(H), None)
    assert rc == L.RB_EINVAL
    assert b"tau" in lib.rb_last_error_string()
    rc = lib.rb_block_1sa(4, 4, 0, None, None, None, 1, 0.5, 7, 1, 1, 1, None, 0, None, None, None, None, None,
                          None, ctypes.byref(H), None)
    assert rc == L.RB_EINVAL
    with pytest.raises(ValueError):
        L.check(L.RB_EINVAL)


@pytest.mark.parametrize("name", ["cfg1_full", "cfg5_s32", "rmat12_t3", "cfg4_s8"])
@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_ranges_partition_permuted_rows(name, precision, world):
    case = load_golden(name)
    rp, bp = case["row_partition"], case["blk_ptr"]
    dp = 64 if precision == "bf16" else 64
    ranges = rbdist.all_ranges(rp, bp, precision, dp, world)
    n = int(rp[-1])
    # contiguous, ordered, covering [0, n) exactly
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    for (b0, e0), (b1, e1) in zip(ranges, ranges[1:]):
        assert e0 == b1 and b0 <= e0
    # cuts fall on work-unit boundaries: block-row starts, or 256-row pair-tile starts of tall rows
    starts = set(rp.tolist())
    for g in range(len(rp) - 1):
        h = rp[g + 1] - rp[g]
        step = 8 if precision == "fp32" else (h if h <= 128 else 256)
        starts.update(range(int(rp[g]), int(rp[g + 1]), int(step)))
    for b, e in ranges:
        assert b in starts or b == n


def test_shard_balance_config_like():
    # 4096 block rows of 64 rows with ~41 blocks each (config-5 shape): shards within one unit of ideal
    rng = np.random.default_rng(0)
    H = 4096
    rp = np.arange(H + 1, dtype=np.int64) * 64
    bp = np.concatenate([[0], np.cumsum(rng.integers(30, 52, H))])
    for world in (2, 4, 8):
        ranges = rbdist.all_ranges(rp, bp, "bf16", 64, world)
        w = np.diff(bp) + 1.0
        loads = [w[b // 64:e // 64].sum() for b, e in ranges]
        assert max(loads) - min(loads) <= 2 * w.max()


def test_csr_validation_messages_match_reference():
    """CsrMatrix.validate raises the reference's messages (matrix.py:79-96), including the first
    offending row for unsorted columns."""
    import pytest

    from paper_2202_05868_b200.types import CsrMatrix

    cases = [(([0, 2, 4, 6], [0, 1, 3, 2, 0, 1]), "row 1: columns not strictly increasing"),
             (([0, 0, 3, 3], [1, 1, 2]), "row 1: columns not strictly increasing"),
             (([0, 3], [2, 1, 0]), "row 0: columns not strictly increasing"),
             (([0, 2], [0, 7]), "column index out of range")]
    for (rp, ci), msg in cases:
        with pytest.raises(ValueError, match=msg):
            CsrMatrix(len(rp) - 1, 4, np.array(rp), np.array(ci), np.ones(len(ci))).validate()

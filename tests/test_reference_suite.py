"""The reference's OWN hot-path test files, run against the drop-in.

tests/reference_shim.py rebinds ``rowblock.block_1sa`` / ``vbr_from_grouping`` / ``spmm_vbr`` (in every
loaded rowblock module) to adapters over this repo's GPU implementations, then pytest runs the
reference's test_blocking.py, test_vbr.py, test_multiply.py, test_metrics.py and test_acceptance.py
(A1–A8, including A5's 50-instance SpMM oracle equivalence at 1e-9 relative, met by the fp64 path)
unchanged.  The installed reference and its test files come from tools/install_reference.sh
(baseline/_ref, git-ignored, shipped to the GPU box with the snapshot); without them the test skips.
The shim's call counts prove the drop-in, not the reference, answered.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "ref_tests")
FILES = ["test_blocking.py", "test_vbr.py", "test_multiply.py", "test_metrics.py", "test_acceptance.py"]


def _have_reference():
    return os.path.isdir(os.path.join(REF, "rowblock")) and all(
        os.path.exists(os.path.join(REF_TESTS, f)) for f in FILES)


@pytest.mark.skipif(not _have_reference(), reason="reference not installed (tools/install_reference.sh)")
def test_reference_suite_against_drop_in(tmp_path):
    counts = tmp_path / "counts.json"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tests"), REF, ROOT]),
               RB_SHIM_COUNTS=str(counts))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "reference_shim", "-p", "no:cacheprovider", "-c",
           os.path.join(REF_TESTS, "pytest.ini"), *FILES]
    r = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=1500)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-40:])
    assert r.returncode == 0, tail
    n = json.loads(counts.read_text())
    assert n["block_1sa"] > 100 and n["vbr_from_grouping"] > 50 and n["spmm_vbr"] > 50, n
    print(tail.splitlines()[-1], n)


@pytest.mark.skipif(not _have_reference(), reason="reference not installed (tools/install_reference.sh)")
def test_drop_in_accepts_reference_objects():
    """Real rowblock objects (CsrMatrix, ColumnPartition, MergePolicy, RowGrouping, VbrMatrix,
    DenseMatrix) go straight into the drop-in; results equal the reference's on the same objects."""
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import rowblock as R

    import paper_2202_05868_b200 as rb

    rng = np.random.default_rng(11)
    keys = rng.choice(300 * 200, size=3000, replace=False)
    A = R.csr_from_triplets(300, 200, [(int(k // 200), int(k % 200), float(v))
                                       for k, v in zip(keys, rng.uniform(0.1, 1.0, len(keys)))])
    q = R.ColumnPartition.uniform(200, 16)
    pol = R.MergePolicy(tau=0.4)
    g_ref = R.block_1sa(A, q, pol)
    g = rb.block_1sa(A, q, pol)
    assert np.array_equal(g.group_of, g_ref.group_of)
    assert [list(x.rows) for x in g.groups] == [list(x.rows) for x in g_ref.groups]
    V_ref = R.vbr_from_grouping(A, g_ref, q)
    V = rb.vbr_from_grouping(A, g_ref, q)  # a reference RowGrouping in
    assert np.array_equal(V.row_perm, V_ref.row_perm) and np.array_equal(V.row_partition, V_ref.row_partition)
    assert [[b.bcol for b in br] for br in V.block_rows] == [[b.bcol for b in br] for br in V_ref.block_rows]
    B = R.DenseMatrix.from_array(rng.random((200, 24)))
    C_ref = R.spmm_vbr(V_ref, B).data
    for VV in (V, V_ref):  # ours, and a reference VbrMatrix (rebuilt on the device from its payloads)
        C = rb.spmm_vbr(VV, B, precision="fp64").data
        nz = C_ref != 0
        assert np.all(np.abs(C - C_ref)[nz] <= 1e-12 * np.abs(C_ref)[nz])
        assert np.array_equal(C[~nz], C_ref[~nz])
        C32 = rb.spmm_vbr(VV, B, precision="fp32").data
        assert np.all(np.abs(C32 - C_ref) <= 1e-5 * (np.abs(A.to_dense()) @ B.data) + 1e-30)

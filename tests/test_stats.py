"""Blocking-quality rows: blocking_stats / verify_density_bound /
blocking_curve / curve_select.

CPU: the oracle's restatement (oracle.group_stats_np) against the reference-generated fixtures
(tests/golden/golden_stats.npz, make_golden_stats.py), and curve_select's host logic.
GPU: the device kernel (rb_group_stats) through the drop-in API, bit-exact integers and
verdicts, floats equal to the reference's (same integer numerators/denominators)."""
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, load_golden, load_golden_small

CASES = ["cfg1_full", "cfg4_s8", "cfg5_s32", "rmat12_t3", "rmat12_t9"]


def golden_stats():
    z = np.load(os.path.join(GOLDEN, "golden_stats.npz"))
    out = {}
    for k in z.files:
        name, key = k.split("__", 1)
        out.setdefault(name, {})[key] = z[k]
    return out


GS = golden_stats()


def all_cases():
    small = load_golden_small()
    for name in sorted(small):
        if name in GS:
            yield name, small[name]
    for name in CASES:
        yield name, load_golden(name)


def check_against(res, ref, name):
    assert np.array_equal(res["stored_cols"], ref["g_stored_cols"]), name
    assert np.array_equal(res["element_nnz"], ref["g_element_nnz"]), name
    assert np.array_equal(res["quotient_nnz"], ref["g_quotient_nnz"]), name
    assert np.array_equal(np.asarray(res["element_ok"], bool), ref["g_element_ok"].astype(bool)), name
    assert np.array_equal(np.asarray(res["quotient_ok"], bool), ref["g_quotient_ok"].astype(bool)), name
    assert res["stored_area"] == int(ref["stored_area"]), name


def test_oracle_group_stats_matches_reference():
    n = 0
    for name, c in all_cases():
        res = oracle.group_stats_np(c["row_ptr"], c["col_idx"], c["boundaries"], c["row_perm"], c["group_ptr"],
                                    c["pattern_ptr"], c["pattern_idx"], float(c["tau"]))
        ref = GS[name]
        check_against(res, ref, name)
        assert res["nnz"] / res["stored_area"] == float(ref["rho_prime"]), name
        if res["n_blocks"]:
            assert res["height_sum"] / res["n_blocks"] == float(ref["delta_h_prime"]), name
        assert res["element_bound"] == float(ref["element_bound"]), name
        n += 1
    assert n > 100


def test_curve_select_host_logic():
    from paper_2202_05868_b200.metrics import BlockingCurve, BlockingStats, curve_select

    c = GS["curve"]
    pts = tuple((float(t), BlockingStats(rho_prime=float(r), delta_h_prime=float(d), n_groups=int(g),
                                         n_stored_blocks=int(b), fill_in=0, nnz=0, stored_area=int(a),
                                         group_mean_height=float(m)))
                for t, r, d, g, b, a, m in zip(c["taus"], c["rho_prime"], c["delta_h_prime"], c["n_groups"],
                                               c["n_stored_blocks"], c["stored_area"], c["group_mean_height"]))
    curve = BlockingCurve(pts, {})
    for h in (1.0, 1.2, 2.0):
        assert curve_select(curve, at_height=h)[0] == float(c[f"select_h_{h}"])
    for d in (0.02, 0.05):
        assert curve_select(curve, at_density=d)[0] == float(c[f"select_d_{d}"])
    with pytest.raises(ValueError):
        curve_select(curve)
    with pytest.raises(ValueError):
        curve_select(curve, at_height=1.0, at_density=0.1)
    with pytest.raises(ValueError):
        curve_select(BlockingCurve((), {}), at_height=1.0)


# ------------------------------------------------------------------------------------------ GPU


def _objects(c):
    import paper_2202_05868_b200 as rb
    from paper_2202_05868_b200.types import RowGroup, RowGrouping

    A = rb.CsrMatrix(int(c["n_rows"]), int(c["n_cols"]), c["row_ptr"], c["col_idx"], c["values"])
    q = rb.ColumnPartition(int(c["n_cols"]), c["boundaries"])
    gp, pp = c["group_ptr"], c["pattern_ptr"]
    groups = [RowGroup(c["row_perm"][gp[g]:gp[g + 1]], c["pattern_idx"][pp[g]:pp[g + 1]], int(c["seed_size"][g]))
              for g in range(len(gp) - 1)]
    return A, q, RowGrouping(c["group_of"], groups)


@pytest.mark.gpu
def test_device_stats_match_reference():
    from paper_2202_05868_b200 import metrics as M

    for name, c in all_cases():
        A, q, G = _objects(c)
        tau = float(c["tau"])
        ref = GS[name]
        s = M.blocking_stats(A, G, q, tau=tau, check_bound=True)
        assert s.stored_area == int(ref["stored_area"]) and s.n_stored_blocks == int(ref["n_stored_blocks"]), name
        assert s.rho_prime == float(ref["rho_prime"]) and s.delta_h_prime == float(ref["delta_h_prime"]), name
        assert s.fill_in == int(ref["fill_in"]) and s.n_groups == int(ref["n_groups"]), name
        assert s.group_mean_height == float(ref["group_mean_height"]), name
        assert s.density_bound_ok == bool(ref["density_bound_ok"]), name
        rep = M.verify_density_bound(A, G, q, tau)
        assert rep.all_ok == bool(ref["density_bound_ok"]), name
        assert rep.element_bound == float(ref["element_bound"]), name
        assert np.array_equal([g.stored_cols for g in rep.groups], ref["g_stored_cols"]), name
        assert np.array_equal([g.quotient_nnz for g in rep.groups], ref["g_quotient_nnz"]), name
        assert np.array_equal([g.element_ok for g in rep.groups], ref["g_element_ok"].astype(bool)), name
        assert np.array_equal([g.element_density for g in rep.groups], ref["g_element_density"]), name


@pytest.mark.gpu
def test_device_curve_matches_reference():
    import paper_2202_05868_b200 as rb
    from paper_2202_05868_b200 import metrics as M

    c = load_golden("cfg1_full")
    A, q, _ = _objects(c)
    ref = GS["curve"]
    curve = M.blocking_curve(A, q, [float(t) for t in ref["taus"]], rb.MergePolicy(tau=0.5))
    assert curve.taus() == [float(t) for t in ref["taus"]]
    for i, (_, s) in enumerate(curve.points):
        assert s.n_groups == int(ref["n_groups"][i]) and s.stored_area == int(ref["stored_area"][i])
        assert s.rho_prime == float(ref["rho_prime"][i]) and s.delta_h_prime == float(ref["delta_h_prime"][i])
        assert s.density_bound_ok == bool(ref["density_bound_ok"][i])
    assert M.curve_select(curve, at_height=1.2)[0] == float(ref["select_h_1.2"])
    # the concurrent form (one host thread per listed device; points sharing a device serialise)
    # gives the same curve; on a 1-GPU box both threads use cuda:0
    par = M.blocking_curve(A, q, [float(t) for t in ref["taus"]], rb.MergePolicy(tau=0.5), jobs=2, devices=[0, 0])
    assert par.taus() == curve.taus() and [s for _, s in par.points] == [s for _, s in curve.points]
    with pytest.raises(ValueError):
        M.blocking_curve(A, q, [0.5, 0.3])
    with pytest.raises(ValueError):
        M.blocking_curve(A, q, [])


@pytest.mark.gpu
def test_device_stats_errors():
    import paper_2202_05868_b200 as rb
    from paper_2202_05868_b200 import metrics as M

    c = load_golden("cfg1_full")
    A, q, G = _objects(c)
    with pytest.raises(ValueError):
        M.blocking_stats(A, G, q, check_bound=True)  # check_bound requires tau
    E = rb.CsrMatrix(3, 4, np.zeros(4, np.int64), np.zeros(0, np.int64), np.zeros(0))
    with pytest.raises(ValueError):
        M.blocking_stats(E, G, rb.ColumnPartition.uniform(4, 2))

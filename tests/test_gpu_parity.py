"""GPU parity: the CUDA path (through the C ABI) against reference-generated golden vectors and the oracle.

Structure (1-SA grouping, VBR block structure, payload reconstruction) must be
bit-exact.  C tolerances (fp32 accumulation, stated here):
  * fp32 check path vs the reference's float64 C:            |err| <= 1e-5 * (|A|·|B|)
  * bf16 / fp16 tensor-core path vs the float64 product of the SAME bf16/fp16-rounded
    inputs (only fp32 accumulation differs):                   |err| <= 1e-4 * (|A|·|B|)
  * bf16 tensor-core path vs the reference on the raw float64 inputs: rel <= 1e-2
    (north_star tolerance) measured as |err| <= 1e-2 * (|A|·|B|)
Rows of A without nonzeros must come out exactly 0.
"""
import numpy as np
import pytest
import torch

import paper_2202_05868_b200 as rb
from conftest import MEDIUM, golden_b, load_golden

pytestmark = pytest.mark.gpu


def csr_of(case):
    return rb.CsrMatrix(int(case["n_rows"]), int(case["n_cols"]), case["row_ptr"], case["col_idx"], case["values"])


def part_of(case):
    return rb.ColumnPartition(int(case["n_cols"]), case["boundaries"])


def policy_of(case):
    return rb.MergePolicy(similarity="cosine" if int(case["cosine"]) else "jaccard", tau=float(case["tau"]),
                          bounded=bool(case["bounded"]), pattern_update=bool(case["pattern_update"]))


def check_grouping(g, case, name=""):
    assert np.array_equal(g.group_of, case["group_of"]), name
    rows = np.concatenate([gr.rows for gr in g.groups]) if g.n_groups else np.zeros(0, np.int64)
    assert np.array_equal(rows, case["row_perm"]), name
    assert np.array_equal(np.concatenate([[0], np.cumsum(g.heights())]), case["row_partition"]), name
    assert np.array_equal(np.array([gr.seed_size for gr in g.groups], np.int64), case["seed_size"]), name
    pats = np.concatenate([gr.pattern for gr in g.groups]) if g.n_groups else np.zeros(0, np.int64)
    assert np.array_equal(pats, case["pattern_idx"]), name
    assert np.array_equal(np.concatenate([[0], np.cumsum([len(gr.pattern) for gr in g.groups])]),
                          case["pattern_ptr"]), name


def check_vbr_structure(V, case, name=""):
    assert np.array_equal(V.row_perm, case["row_perm"]), name
    assert np.array_equal(V.row_partition, case["row_partition"]), name
    rp, bp, bc = V.device.host_structure()
    assert np.array_equal(bp, case["blk_ptr"]), name
    assert np.array_equal(bc, case["blk_col"]), name
    assert V.stored_area == int(case["stored_area"]), name


def vbr_to_dense(V):
    out = np.zeros((V.n_rows, V.n_cols))
    b = V.col_partition.boundaries
    for g in range(V.n_block_rows):
        rows = V.row_perm[V.row_partition[g]:V.row_partition[g + 1]]
        for blk in V.block_rows[g]:
            out[rows, b[blk.bcol]:b[blk.bcol + 1]] = blk.data
    return out


def rounded(x, dt):
    """Correctly rounded (RNE) float64 -> dt -> float64, as the device's __double2bfloat16 /
    __double2half do (torch's .to(bfloat16) rounds twice, via float32)."""
    x = np.asarray(x, np.float64)
    if dt == torch.float16:
        return x.astype(np.float16).astype(np.float64)
    b = np.ascontiguousarray(x).view(np.uint64)
    lsb = (b >> np.uint64(45)) & np.uint64(1)
    r = (b + np.uint64((1 << 44) - 1) + lsb) & ~np.uint64((1 << 45) - 1)
    return r.view(np.float64)


def dense_of(case, dt=None):
    A = np.zeros((int(case["n_rows"]), int(case["n_cols"])))
    rows = np.repeat(np.arange(int(case["n_rows"])), np.diff(case["row_ptr"]))
    vals = case["values"] if dt is None else rounded(case["values"], dt)
    A[rows, case["col_idx"]] = vals
    return A


def assert_close(C, ref, bound, rtol, name=""):
    err = np.abs(C - ref)
    assert np.all(err <= rtol * bound + 1e-30), f"{name}: max scaled err {np.max(err / (bound + 1e-30)):.3e}"


# ------------------------------------------------------------------ 1-SA + VBR structure


def test_block_1sa_bit_exact_golden_small(golden_small):
    for name, case in golden_small.items():
        g = rb.block_1sa(csr_of(case), part_of(case), policy_of(case), bool(case["use_compression"]))
        check_grouping(g, case, name)


def test_vbr_structure_and_reconstruction_golden_small(golden_small):
    for name, case in golden_small.items():
        A = csr_of(case)
        q = part_of(case)
        g = rb.block_1sa(A, q, policy_of(case), bool(case["use_compression"]))
        V = rb.vbr_from_grouping(A, g, q)
        check_vbr_structure(V, case, name)
        assert np.array_equal(vbr_to_dense(V), A.to_dense()), name  # bit-exact (test_vbr.py:73-88)


@pytest.mark.parametrize("name", MEDIUM)
def test_block_1sa_and_vbr_medium(name):
    case = load_golden(name)
    A, q = csr_of(case), part_of(case)
    g = rb.block_1sa(A, q, policy_of(case), bool(case["use_compression"]))
    check_grouping(g, case, name)
    V = rb.vbr_from_grouping(A, g, q)
    check_vbr_structure(V, case, name)


# ------------------------------------------------------------------ SpMM


@pytest.mark.parametrize("precision", ["fp32", "bf16", "fp16"])
def test_spmm_golden_small(golden_small, precision):
    tdt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": None}[precision]
    n_checked = 0
    for name, case in golden_small.items():
        B = golden_b(case)
        if B is None or "C" not in case:
            continue
        A, q = csr_of(case), part_of(case)
        V = rb.vbr_from_grouping(A, rb.block_1sa(A, q, policy_of(case), bool(case["use_compression"])), q)
        C = rb.spmm_vbr(V, rb.DenseMatrix.from_array(B), precision=precision).data
        Ad = dense_of(case)
        bound = np.abs(Ad) @ np.abs(B)
        if precision == "fp32":
            assert_close(C, case["C"], bound, 1e-5, name)
        else:
            ref_r = dense_of(case, tdt) @ rounded(B, tdt)
            assert_close(C, ref_r, np.abs(dense_of(case, tdt)) @ np.abs(rounded(B, tdt)), 1e-4, name)
            if precision == "bf16":
                assert_close(C, case["C"], bound, 1e-2, name)
        empty = np.diff(case["row_ptr"]) == 0
        assert np.all(C[empty] == 0.0), name
        n_checked += 1
    assert n_checked > 100


@pytest.mark.parametrize("name", ["cfg1_full", "cfg4_s8", "cfg5_s32", "rmat12_t3", "rmat12_t9", "rmat16_t7"])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_spmm_medium_checksums(name, precision):
    """C of the reference's spmm_vbr (multiply.py:72-97) pinned by two checksums per row (C·r and
    the row sums) recorded when the golden case was made; the R-MAT cases run the skinny kernels
    on power-law input (config 3's shape)."""
    import scipy.sparse as sp

    case = load_golden(name)
    B = golden_b(case)
    A, q = csr_of(case), part_of(case)
    V = rb.vbr_from_grouping(A, rb.block_1sa(A, q, policy_of(case), True), q)
    C = rb.spmm_vbr(V, rb.DenseMatrix.from_array(B), precision=precision).data
    r = np.random.default_rng(7).standard_normal(B.shape[1])
    tol = 1e-5 if precision == "fp32" else 1e-2
    Aabs = sp.csr_matrix((np.abs(A.values), A.col_idx, A.row_ptr), shape=(A.n_rows, A.n_cols))
    AB = Aabs @ np.abs(B)
    assert np.all(np.abs(C @ r - case["C_dot_r"]) <= tol * (AB @ np.abs(r)) + 1e-12)
    assert np.all(np.abs(C.sum(axis=1) - case["C_rowsum"]) <= tol * AB.sum(1) + 1e-12)
    empty = np.diff(A.row_ptr) == 0
    assert np.all(C[empty] == 0.0)


def test_spmm_tall_and_short_shapes_bf16():
    """Exercise both tensor-core kernels: tall block rows (h > 128, several M-tiles, ragged last
    tile), short block rows of every padded height (16/32/64/128), N not a multiple of 64,
    Δ > 64 (two K chunks per block), ragged last segment."""
    rng = np.random.default_rng(5)
    heights = [1, 3, 16, 17, 40, 64, 100, 128, 129, 300, 513]
    n_cols, delta, N = 1000, 96, 200
    rows, cols = [], []
    r0 = 0
    for h in heights:
        segs = rng.choice((n_cols + delta - 1) // delta, size=int(rng.integers(1, 6)), replace=False)
        for s in segs:
            lo, hi = s * delta, min(n_cols, (s + 1) * delta)
            for r in range(r0, r0 + h):
                c = rng.choice(np.arange(lo, hi), size=max(1, (hi - lo) // 5), replace=False)
                rows.append(np.full(len(c), r))
                cols.append(c)
        r0 += h
    n_rows = r0
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    vals = rounded(rng.uniform(-1, 1, len(rows)), torch.bfloat16)
    keep = vals != 0
    from paper_2202_05868_b200.types import csr_from_coo
    A = csr_from_coo(n_rows, n_cols, rows[keep], cols[keep], vals[keep], sum_duplicates=True)
    perm = rng.permutation(n_rows)  # groups by construction, rows scrambled inside the grouping
    q = rb.ColumnPartition.uniform(n_cols, delta)
    groups, start = [], 0
    from paper_2202_05868_b200.types import RowGroup, RowGrouping
    go = np.zeros(n_rows, np.int64)
    for gi, h in enumerate(heights):
        members = np.arange(start, start + h)
        go[members] = gi
        groups.append(RowGroup(members, np.zeros(0), 0))
        start += h
    G = RowGrouping(go, groups)
    V = rb.vbr_from_grouping(A, G, q)
    B = rounded(rng.uniform(-1, 1, (n_cols, N)), torch.bfloat16)
    C = rb.spmm_vbr(V, rb.DenseMatrix.from_array(B), precision="bf16").data
    ref = A.to_dense() @ B
    assert_close(C, ref, np.abs(A.to_dense()) @ np.abs(B), 1e-4, "shapes")
    del perm


@pytest.mark.parametrize("h,delta,N,delay", [(64, 64, 1024, "8"), (40, 96, 320, "0"), (16, 64, 200, "3"),
                                              (100, 64, 256, "8")])
def test_spmm_sweep_kernel(h, delta, N, delay, monkeypatch):
    """spmm_sweep_kernel (multi-slot circular sweep of one short height class): many block rows of
    height h with random block columns, forced on (RB_SWEEP=2) so that small cases use it; two K
    chunks per block when Δ > 64, a ragged last column slab when N % 256 != 0, slot reuse with and
    without a delay.  C against the float64 product of the same rounded inputs; run-to-run identical."""
    monkeypatch.setenv("RB_SWEEP", "2")
    monkeypatch.setenv("RB_SWEEP_DELAY", delay)
    rng = np.random.default_rng(h + N)
    n_groups, n_seg = 300, 48
    n_cols = n_seg * delta
    rows, cols = [], []
    for gi in range(n_groups):
        segs = rng.choice(n_seg, size=int(rng.integers(1, 12)), replace=False)
        for sgi in segs:
            for r in range(gi * h, (gi + 1) * h):
                c = rng.choice(np.arange(sgi * delta, (sgi + 1) * delta), size=int(rng.integers(1, 8)), replace=False)
                rows.append(np.full(len(c), r))
                cols.append(c)
    n_rows = n_groups * h
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    vals = rounded(rng.uniform(-1, 1, len(rows)), torch.bfloat16)
    keep = vals != 0
    from paper_2202_05868_b200.types import RowGroup, RowGrouping, csr_from_coo
    perm = rng.permutation(n_rows)
    go = np.zeros(n_rows, np.int64)
    groups = []
    for gi in range(n_groups):
        members = np.sort(perm[gi * h:(gi + 1) * h])
        go[members] = gi
        groups.append(RowGroup(members, np.zeros(0), 0))
    # scramble the rows of A consistently with the grouping: row perm[i] of the grouping is row i of A
    A = csr_from_coo(n_rows, n_cols, perm[rows[keep]], cols[keep], vals[keep], sum_duplicates=True)
    V = rb.vbr_from_grouping(A, RowGrouping(go, groups), rb.ColumnPartition.uniform(n_cols, delta))
    info = V.device.plan_info(N, "bf16")
    assert info["n_sweep_steps"] > 0 and info["sweep_slots"] == min(16, 512 // (2 * max(16, 1 << (h - 1).bit_length())))
    B = rounded(rng.uniform(-1, 1, (n_cols, N)), torch.bfloat16)
    C = rb.spmm_vbr(V, rb.DenseMatrix.from_array(B), precision="bf16").data
    Ad = A.to_dense()
    assert_close(C, Ad @ B, np.abs(Ad) @ np.abs(B), 1e-4, "sweep")
    C2 = rb.spmm_vbr(V, rb.DenseMatrix.from_array(B), precision="bf16").data
    assert np.array_equal(C, C2)


@pytest.mark.parametrize("variant", [("RB_SWEEP_PAIR", "1"), ("RB_SWEEP_BIG", "0"), ("RB_SWEEP_DELAY", "20")])
@pytest.mark.parametrize("precision", ["bf16", "fp16"])
def test_spmm_sweep_kernel_variants(variant, precision, monkeypatch):
    """The sweep kernel's stage-ring variants (pair barriers, 5 x 40 KB ring, long slot delay) and
    fp16 operands on config 5's shape (h = 64, N = 1024 -> 4 slabs), forced on a small matrix."""
    monkeypatch.setenv("RB_SWEEP", "2")
    monkeypatch.setenv(*variant)
    rng = np.random.default_rng(hash(variant) % 1000)
    n_groups, h, delta, n_seg, N = 160, 64, 64, 40, 1024
    from paper_2202_05868_b200.types import RowGroup, RowGrouping, csr_from_coo
    rows, cols = [], []
    for gi in range(n_groups):
        for sgi in rng.choice(n_seg, size=int(rng.integers(1, 8)), replace=False):
            for r in range(gi * h, (gi + 1) * h):
                c = rng.choice(np.arange(sgi * delta, (sgi + 1) * delta), size=int(rng.integers(1, 6)), replace=False)
                rows.append(np.full(len(c), r))
                cols.append(c)
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    tdt = torch.float16 if precision == "fp16" else torch.bfloat16
    vals = rounded(rng.uniform(-1, 1, len(rows)), tdt)
    keep = vals != 0
    A = csr_from_coo(n_groups * h, n_seg * delta, rows[keep], cols[keep], vals[keep], sum_duplicates=True)
    go = np.repeat(np.arange(n_groups), h)
    G = RowGrouping(go, [RowGroup(np.arange(g * h, (g + 1) * h), np.zeros(0), 0) for g in range(n_groups)])
    V = rb.vbr_from_grouping(A, G, rb.ColumnPartition.uniform(n_seg * delta, delta))
    B = rounded(rng.uniform(-1, 1, (n_seg * delta, N)), tdt)
    assert V.device.plan_info(N, precision)["n_sweep_steps"] > 0
    C = rb.spmm_vbr(V, rb.DenseMatrix.from_array(B), precision=precision).data
    Ad = A.to_dense()
    assert_close(C, Ad @ B, np.abs(Ad) @ np.abs(B), 1e-4, str(variant))


@pytest.mark.parametrize("name", ["rmat12_t3", "rmat16_t7", "cfg1_full"])
@pytest.mark.parametrize("precision", ["bf16", "fp16", "fp32"])
def test_compact_payloads_match_tiles(name, precision, monkeypatch):
    """Skinny block rows multiplied from compact payloads (default) and from their padded tiles
    (RB_COMPACT_H=0): both within the stated tolerance of the float64 product of the same rounded
    inputs, the compact run launching the CSR engine and no tile skinny kernel."""
    import scipy.sparse as sp
    from paper_2202_05868_b200 import config

    case = load_golden(name)
    A, q = csr_of(case), part_of(case)
    B = golden_b(case)
    tdt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}[precision]
    Ar = sp.csr_matrix((rounded(A.values, tdt) if precision != "fp32" else A.values.astype(np.float32).astype(np.float64),
                        A.col_idx, A.row_ptr), shape=(A.n_rows, A.n_cols))
    Br = rounded(B, tdt) if precision != "fp32" else B.astype(np.float32).astype(np.float64)
    ref = Ar @ Br
    bound = abs(Ar) @ np.abs(Br)
    out = {}
    for h in (8, 0):
        monkeypatch.setattr(config, "_COMPACT_H", h)
        V = rb.vbr_from_grouping(A, rb.block_1sa(A, q, policy_of(case), True), q)
        out[h] = rb.spmm_vbr(V, rb.DenseMatrix.from_array(B), precision=precision).data
        assert_close(out[h], ref, bound, 1e-5 if precision == "fp32" else 1e-4, f"{name} compact_h={h}")
    empty = np.diff(A.row_ptr) == 0
    assert np.all(out[8][empty] == 0.0)


def test_shard_sub_vbrs_assemble_full_product():
    """bench.py --gpus N's per-rank path on one GPU: every rank's sub-VBR (dist.shard_vbr, own tiles)
    computes its rows in permuted order; placed at row_perm they equal the single-GPU product."""
    from paper_2202_05868_b200 import dist as rbdist
    from paper_2202_05868_b200.device import DeviceCsr, block_1sa_device
    from paper_2202_05868_b200.types import MergePolicy

    for name in ("cfg5_s32", "cfg4_s8", "rmat12_t3"):
        case = load_golden(name)
        A, q = csr_of(case), part_of(case)
        dA = DeviceCsr.from_host(A)
        dg = block_1sa_device(dA, q, MergePolicy(tau=float(case["tau"])), True)
        B = torch.from_numpy(golden_b(case)).to(torch.bfloat16).cuda()
        full = rb.vbr_from_grouping(A, rb.block_1sa(A, q, policy_of(case), True), q).device.spmm(B, precision="bf16")
        perm = dg.row_perm[: A.n_rows].to(torch.int64)
        for world in (2, 3, 8):
            C = torch.full_like(full, float("nan"))
            for k in range(world):
                dv, (b, e), _ = rbdist.shard_vbr(dA, q, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], "bf16", k, world)
                assert dv.n_rows == e - b
                if e > b:
                    C[perm[b:e]] = dv.spmm(B, precision="bf16")
            torch.cuda.synchronize()
            assert not torch.isnan(C).any(), (name, world)
            err = (C.double() - full.double()).abs().max().item()
            assert err <= 1e-5 * max(1.0, full.abs().max().item()), (name, world, err)


def test_spmm_medium_cfg5_through_sweep(monkeypatch):
    """The reference-generated 1/32-scale config 5 (128 block rows of h = 64) through the sweep kernel."""
    monkeypatch.setenv("RB_SWEEP", "2")
    case = load_golden("cfg5_s32")
    A, q = csr_of(case), part_of(case)
    V = rb.vbr_from_grouping(A, rb.block_1sa(A, q, policy_of(case), True), q)
    assert V.device.plan_info(int(case["B_shape"][1]), "bf16")["n_sweep_steps"] > 0
    test_spmm_medium_checksums("cfg5_s32", "bf16")


def test_spmm_device_api_and_determinism():
    rng = np.random.default_rng(9)
    case = load_golden("cfg5_s32")
    A, q = csr_of(case), part_of(case)
    V = rb.vbr_from_grouping(A, rb.block_1sa(A, q, policy_of(case), True), q)
    B = torch.rand((A.n_cols, 256), device="cuda").to(torch.bfloat16)
    C1 = rb.spmm_vbr_device(V, B)
    C2 = rb.spmm_vbr_device(V, B)
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)  # bit-identical run to run
    ref = torch.from_numpy(A.to_dense()).cuda().to(torch.bfloat16).double() @ B.double()
    err = (C1.double() - ref).abs().max().item()
    assert err <= 1e-4 * ref.abs().max().item()
    del rng


@pytest.mark.parametrize("name,N,split", [("rmat12_t3", 64, None), ("cfg5_s32", 256, None), ("cfg4_s8", 512, "2")])
def test_one_plan_on_two_streams(name, N, split, monkeypatch):
    """One DeviceVbr (one cached plan per N) driven from two streams and two host threads at once:
    the plan's self-resetting work counters and split partials (skinny scheduler, split hub rows,
    tall split-K tail) must not be shared by overlapping executions (rowblock_b200.h: executions
    of one plan are serialised on the device).  Each result equals the single-stream result."""
    import threading

    if split:
        monkeypatch.setenv("RB_TALL_SPLIT", split)
    case = load_golden(name)
    A, q = csr_of(case), part_of(case)
    V = rb.vbr_from_grouping(A, rb.block_1sa(A, q, policy_of(case), True), q)
    dv = V.device
    g = torch.Generator(device="cuda").manual_seed(5)
    Bs = [torch.rand((A.n_cols, N), device="cuda", generator=g).to(torch.bfloat16) for _ in range(4)]
    refs = [dv.spmm(B, precision="bf16").clone() for B in Bs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = [torch.empty_like(r) for r in refs]
    for rep in range(3):
        for k, B in enumerate(Bs):  # alternate streams without host synchronisation
            st = streams[k % 2]
            with torch.cuda.stream(st):
                dv.spmm(B, out=outs[k], precision="bf16", stream=st)
        torch.cuda.synchronize()
        for k in range(len(Bs)):
            assert torch.equal(outs[k], refs[k]), (rep, k)
    # two host threads, each on its own stream
    errs = []

    def worker(k):
        try:
            st = streams[k % 2]
            with torch.cuda.stream(st):
                for _ in range(4):
                    dv.spmm(Bs[k], out=outs[k], precision="bf16", stream=st)
            st.synchronize()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ths = [threading.Thread(target=worker, args=(k,)) for k in range(len(Bs))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    torch.cuda.synchronize()
    assert not errs
    for k in range(len(Bs)):
        assert torch.equal(outs[k], refs[k]), k


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_nonfinite_b_raises(bad):
    """The reference propagates NaN / Inf of B through its dense block payloads (multiply.py:89);
    the GPU path skips zero tile entries and pads tiles, so it cannot reproduce that pattern and
    raises ValueError instead of returning a different one (spmm_vbr and spmm_vbr_many)."""
    case = load_golden("cfg1_full")
    A, q = csr_of(case), part_of(case)
    V = rb.vbr_from_grouping(A, rb.block_1sa(A, q, policy_of(case), True), q)
    B = np.random.default_rng(3).random((A.n_cols, 32))
    B[17, 5] = bad
    for prec in ("bf16", "fp32"):
        with pytest.raises(ValueError, match="NaN or Inf"):
            rb.spmm_vbr(V, rb.DenseMatrix.from_array(B), precision=prec)
    ok = np.random.default_rng(4).random((A.n_cols, 32))
    with pytest.raises(ValueError, match="NaN or Inf"):
        rb.spmm_vbr_many(V, [rb.DenseMatrix.from_array(ok), rb.DenseMatrix.from_array(B)], precision="bf16")
    C = rb.spmm_vbr(V, rb.DenseMatrix.from_array(ok), precision="bf16").data  # finite B still works
    assert np.isfinite(C).all()


def test_errors_map_to_reference_exceptions():
    A = rb.csr_from_triplets(4, 6, [(0, 0, 1.0), (0, 1, 1.0), (1, 3, 1.0), (2, 2, 1.0), (3, 4, 1.0), (3, 5, 1.0)])
    q = rb.ColumnPartition.uniform(6, 3)
    g = rb.block_1sa(A, q, rb.MergePolicy(tau=0.5))
    with pytest.raises(ValueError):
        rb.vbr_from_grouping(A, g, rb.ColumnPartition.uniform(5, 3))
    V = rb.vbr_from_grouping(A, g, q)
    with pytest.raises(ValueError):
        rb.spmm_vbr(V, rb.DenseMatrix.zeros(5, 2))
    with pytest.raises(ValueError):
        rb.MergePolicy(tau=1.5)


@pytest.fixture
def force_sparse_1sa(monkeypatch):
    monkeypatch.setenv("RB_1SA_MODE", "sparse")


def test_block_1sa_sparse_path_bit_exact_golden(golden_small, force_sparse_1sa):
    """The inverted-index (pruned) greedy used for large W is exact on every golden case."""
    for name, case in golden_small.items():
        g = rb.block_1sa(csr_of(case), part_of(case), policy_of(case), bool(case["use_compression"]))
        check_grouping(g, case, name)


@pytest.mark.parametrize("name", MEDIUM)
def test_block_1sa_sparse_path_medium(name, force_sparse_1sa):
    case = load_golden(name)
    g = rb.block_1sa(csr_of(case), part_of(case), policy_of(case), bool(case["use_compression"]))
    check_grouping(g, case, name)


@pytest.mark.parametrize("split", ["2", "1"])
def test_spmm_tall_split_k_tail(split, monkeypatch):
    """Tall block rows whose last wave is split along K (partials reduced by the last-arriving
    epilogue warp, in split order): C within the bf16 tolerance, bit-identical run to run (the
    arrival counters reset themselves), and RB_TALL_SPLIT=1 (no split) agrees to tolerance."""
    from paper_2202_05868_b200.device import DeviceCsr, DeviceVbr
    from paper_2202_05868_b200.types import csr_from_coo

    monkeypatch.setenv("RB_TALL_SPLIT", split)
    rng = np.random.default_rng(11)
    heights = [300, 257, 520]  # 2 + 2 + 3 pair tiles (256 rows each)
    n_cols, delta, N = 16384, 64, 300  # 256 segments -> 256 K steps per item; 2 N chunks (second ragged)
    rows, cols, r0 = [], [], 0
    for h in heights:
        nnz = h * 40
        rows.append(r0 + rng.integers(0, h, nnz))
        cols.append(rng.integers(0, n_cols, nnz))
        r0 += h
    keys = np.unique(np.concatenate(rows) * n_cols + np.concatenate(cols))
    vals = rounded(rng.uniform(0.1, 1.0, len(keys)), torch.bfloat16) * rng.choice([-1.0, 1.0], len(keys))
    A = csr_from_coo(r0, n_cols, keys // n_cols, keys % n_cols, vals)
    perm = torch.from_numpy(rng.permutation(r0)).cuda()
    rp = torch.tensor(np.concatenate([[0], np.cumsum(heights)]), device="cuda")
    q = rb.ColumnPartition.uniform(n_cols, delta)
    dv = DeviceVbr.build(DeviceCsr.from_host(A, "cuda"), q, perm, rp, dtypes=("bf16",))
    info = dv.plan_info(N, "bf16")
    n_items = (2 + 2 + 3) * 2
    if split == "1":
        assert info["n_items_tall"] == n_items
    else:
        assert info["n_items_tall"] > n_items  # the tail was split
    B = rounded(rng.uniform(-1, 1, (n_cols, N)), torch.bfloat16)
    Bd = torch.zeros((n_cols, 304), dtype=torch.bfloat16, device="cuda")[:, :N]  # 16-byte row stride
    Bd.copy_(torch.from_numpy(B))
    C1 = dv.spmm(Bd)
    C2 = dv.spmm(Bd)
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)
    Ad = A.to_dense()
    assert_close(C1.cpu().numpy().astype(np.float64), Ad @ B, np.abs(Ad) @ np.abs(B), 1e-4, f"split={split}")


def _grouped_matrix(rng, heights, n_cols, delta, density):
    """A matrix whose block rows are given (heights), scrambled rows, ragged last segment."""
    from paper_2202_05868_b200.types import csr_from_coo

    n_rows = int(sum(heights))
    keys = np.unique(rng.choice(n_rows * n_cols, size=int(density * n_rows * n_cols), replace=False))
    vals = rounded(rng.uniform(0.1, 1.0, len(keys)), torch.bfloat16) * rng.choice([-1.0, 1.0], len(keys))
    A = csr_from_coo(n_rows, n_cols, keys // n_cols, keys % n_cols, vals)
    perm = torch.from_numpy(rng.permutation(n_rows)).cuda()
    rp = torch.tensor(np.concatenate([[0], np.cumsum(heights)]), device="cuda")
    return A, perm, rp


@pytest.mark.parametrize("precision,N,ld", [("fp32", 37, 37), ("fp32", 256, 256), ("bf16", 100, 104),
                                            ("bf16", 300, 304), ("fp16", 64, 64)])
def test_spmm_skinny_block_rows(precision, N, ld, monkeypatch):
    """Block rows with h <= 8 run on the CUDA-core skinny kernel (every height class, lane groups of
    16 and 32, unaligned fp32 B rows, ragged N, empty block rows).  C within tolerance of the
    float64 product of the same rounded inputs; on the fp32 path within 1e-6 of the dense-tile
    SIMT kernel (RB_SKINNY_H=0): skipped terms are exact zeros, but block rows may be cut into parts
    summed separately (small classes are split for parallelism), which reorders the fp32 sums."""
    from paper_2202_05868_b200 import _lib as L
    from paper_2202_05868_b200.device import DeviceCsr, DeviceVbr

    rng = np.random.default_rng(23)
    heights = [1, 2, 3, 4, 5, 8, 1, 1, 7, 2] * 6 + [40, 200]
    A, perm, rp = _grouped_matrix(rng, heights, 700, 48, 0.03)
    q = rb.ColumnPartition.uniform(700, 48)
    dt = L.TORCH_DTYPE[L.PRECISION[precision]]
    Bh = rounded(rng.uniform(-1, 1, (700, N)), dt if dt != torch.float32 else torch.bfloat16)
    Bd = torch.zeros((700, ld), dtype=dt, device="cuda")[:, :N]
    Bd.copy_(torch.from_numpy(Bh))
    Cs = {}
    for sk in ["8", "0"]:
        monkeypatch.setenv("RB_SKINNY_H", sk)
        dv = DeviceVbr.build(DeviceCsr.from_host(A, "cuda"), q, perm, rp, dtypes=(precision,))
        info = dv.plan_info(N, precision)
        assert (info["n_items_skinny"] > 0) == (sk == "8")
        Cs[sk] = dv.spmm(Bd, precision=precision)
        torch.cuda.synchronize()
        assert torch.equal(Cs[sk], dv.spmm(Bd, precision=precision))
    Ad = dense_of({"n_rows": A.n_rows, "n_cols": A.n_cols, "row_ptr": A.row_ptr, "col_idx": A.col_idx,
                   "values": A.values}, None if precision != "fp16" else torch.float16)
    ref = Ad @ Bh
    bound = np.abs(Ad) @ np.abs(Bh)
    tol = 1e-5 if precision == "fp32" else 1e-4
    assert_close(Cs["8"].cpu().numpy().astype(np.float64), ref, bound, tol, f"skinny {precision}")
    if precision == "fp32":
        assert_close(Cs["8"].cpu().numpy().astype(np.float64), Cs["0"].cpu().numpy().astype(np.float64), bound,
                     1e-6, "skinny vs simt")
    else:
        assert_close(Cs["0"].cpu().numpy().astype(np.float64), ref, bound, tol, f"tensor {precision}")


@pytest.mark.parametrize("precision,N", [("fp32", 256), ("bf16", 128), ("bf16", 520)])
def test_spmm_skinny_split_rows(precision, N):
    """Skinny block rows with more than 256 stored blocks (power-law hubs) are cut into parts whose
    partials are summed in part order by the last-arriving part: C within tolerance and
    bit-identical run to run (the arrival counters reset themselves between launches)."""
    from paper_2202_05868_b200 import _lib as L
    from paper_2202_05868_b200.device import DeviceCsr, DeviceVbr
    from paper_2202_05868_b200.types import csr_from_coo

    rng = np.random.default_rng(29)
    n_cols, delta = 40000, 64
    heights = [1, 1, 3, 1, 8, 2, 1]
    per_row = [3000, 40, 900, 1200, 500, 2500, 5]
    rows, cols, r0 = [], [], 0
    for h, k in zip(heights, per_row):
        for r in range(r0, r0 + h):
            c = rng.choice(n_cols, size=k, replace=False)
            rows.append(np.full(k, r))
            cols.append(c)
        r0 += h
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    vals = rounded(rng.uniform(0.1, 1.0, len(rows)), torch.bfloat16) * rng.choice([-1.0, 1.0], len(rows))
    A = csr_from_coo(r0, n_cols, rows, cols, vals)
    perm = torch.from_numpy(rng.permutation(r0)).cuda()
    rp = torch.tensor(np.concatenate([[0], np.cumsum(heights)]), device="cuda")
    q = rb.ColumnPartition.uniform(n_cols, delta)
    dv = DeviceVbr.build(DeviceCsr.from_host(A, "cuda"), q, perm, rp, dtypes=(precision,))
    _, bp, _ = dv.host_structure()
    assert np.diff(bp).max() > 512  # several parts
    dt = L.TORCH_DTYPE[L.PRECISION[precision]]
    Bh = rounded(rng.uniform(-1, 1, (n_cols, N)), torch.bfloat16)
    Bd = torch.from_numpy(Bh).cuda().to(dt)
    C1 = dv.spmm(Bd, precision=precision)
    C2 = dv.spmm(Bd, precision=precision)
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)
    Ad = A.to_dense()
    tol = 1e-5 if precision == "fp32" else 1e-4
    assert_close(C1.cpu().numpy().astype(np.float64), Ad @ Bh, np.abs(Ad) @ np.abs(Bh), tol, "split rows")


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
def test_spmm_vbr_many_pipeline_matches_single(precision):
    """The pipelined multi-RHS API (3 streams, double-buffered) returns, for every B_k, exactly
    what spmm_vbr returns for that B alone (same plan, same kernels), in order."""
    case = load_golden("cfg5_s32")
    A, q = csr_of(case), part_of(case)
    V = rb.vbr_from_grouping(A, rb.block_1sa(A, q, policy_of(case), True), q)
    rng = np.random.default_rng(31)
    Bs = [rb.DenseMatrix.from_array(rng.random((A.n_cols, 96))) for _ in range(5)]
    many = rb.spmm_vbr_many(V, Bs, precision=precision)
    assert len(many) == 5
    for B, C in zip(Bs, many):
        assert np.array_equal(C.data, rb.spmm_vbr(V, B, precision=precision).data)


# ------------------------------------------------------------------ spmm_csr comparator


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_spmm_csr_golden_small(golden_small, precision):
    """spmm_csr on the GPU against the reference's C (spmm_vbr == spmm_csr to 1e-9 in the
    reference, test_acceptance.py:200-205): fp32 within 1e-5, bf16 within 1e-4 of the product of
    the same rounded inputs; empty rows exactly 0."""
    n_checked = 0
    for name, case in golden_small.items():
        B = golden_b(case)
        if B is None or "C" not in case:
            continue
        A = csr_of(case)
        C = rb.spmm_csr(A, rb.DenseMatrix.from_array(B), precision=precision).data
        if precision == "fp32":
            assert_close(C, case["C"], np.abs(dense_of(case)) @ np.abs(B), 1e-5, name)
        else:
            Ar, Br = dense_of(case, torch.bfloat16), rounded(B, torch.bfloat16)
            assert_close(C, Ar @ Br, np.abs(Ar) @ np.abs(Br), 1e-4, name)
        assert np.all(C[np.diff(case["row_ptr"]) == 0] == 0.0), name
        n_checked += 1
    assert n_checked > 100


@pytest.mark.parametrize("precision,N", [("bf16", 128), ("bf16", 300), ("fp32", 70)])
def test_spmm_csr_hub_rows_and_determinism(precision, N):
    """Rows longer than 2048 nonzeros are split into parts reduced in part order; results are
    bit-identical run to run; the device API and the drop-in agree."""
    from paper_2202_05868_b200.device import DeviceCsr
    from paper_2202_05868_b200.types import csr_from_coo

    rng = np.random.default_rng(41)
    n_rows, n_cols = 300, 9000
    per_row = rng.integers(0, 40, n_rows)
    per_row[[3, 100, 299]] = [9000, 5000, 2049]
    rows = np.concatenate([np.full(k, r) for r, k in enumerate(per_row)])
    cols = np.concatenate([rng.choice(n_cols, size=k, replace=False) for k in per_row])
    vals = rounded(rng.uniform(0.1, 1.0, len(rows)), torch.bfloat16) * rng.choice([-1.0, 1.0], len(rows))
    A = csr_from_coo(n_rows, n_cols, rows, cols, vals)
    Bh = rounded(rng.uniform(-1, 1, (n_cols, N)), torch.bfloat16)
    C = rb.spmm_csr(A, rb.DenseMatrix.from_array(Bh), precision=precision).data
    Ad = A.to_dense()
    tol = 1e-5 if precision == "fp32" else 1e-4
    assert_close(C, Ad @ Bh, np.abs(Ad) @ np.abs(Bh), tol, "csr hub rows")
    dA = DeviceCsr.from_host(A, "cuda")
    dt = torch.float32 if precision == "fp32" else torch.bfloat16
    ld = (N + 7) // 8 * 8
    Bd = torch.zeros((n_cols, ld), dtype=dt, device="cuda")[:, :N]
    Bd.copy_(torch.from_numpy(Bh))
    C1, C2 = dA.spmm(Bd, precision=precision), dA.spmm(Bd, precision=precision)
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)
    assert np.array_equal(C1.double().cpu().numpy(), C)


@pytest.mark.parametrize("N", [128, 512])
def test_spmm_csr_uniform_rows_chunked_claims(N):
    """Uniform work lists with many items per resident group are claimed two items per atomic
    (csr_claim_chunk).  An odd item count puts the last claim half past the end.  Every row must
    be written once and equal the product; the result must be bit-identical run to run."""
    from paper_2202_05868_b200.device import DeviceCsr
    from paper_2202_05868_b200.types import csr_from_coo

    rng = np.random.default_rng(53 + N)
    n_rows, n_cols, k = 160001, 2048, 6  # N=128: 160001 items; N=512: 2 slabs each
    rows = np.repeat(np.arange(n_rows), k)
    cols = np.concatenate([rng.choice(n_cols, size=k, replace=False) for _ in range(n_rows)])
    vals = rounded(rng.uniform(-1.0, 1.0, len(rows)), torch.bfloat16)
    A = csr_from_coo(n_rows, n_cols, rows, cols, vals)
    Bh = rounded(rng.uniform(-1, 1, (n_cols, N)), torch.bfloat16)
    dA = DeviceCsr.from_host(A, "cuda")
    Bd = torch.from_numpy(Bh).to(torch.bfloat16).cuda()
    C1, C2 = dA.spmm(Bd, precision="bf16"), dA.spmm(Bd, precision="bf16")
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)
    Ad = torch.sparse_csr_tensor(torch.from_numpy(A.row_ptr), torch.from_numpy(A.col_idx), torch.from_numpy(A.values),
                                 size=(n_rows, n_cols))
    ref = (Ad @ torch.from_numpy(Bh)).numpy()
    bound = np.abs(A.values).max() * k * np.abs(Bh).max()
    assert np.abs(C1.double().cpu().numpy() - ref).max() <= 1e-4 * bound


def test_edge_shapes_through_the_drop_in():
    """Degenerate inputs behave as in the reference: an all-zero matrix (every row its own empty
    block row or one empty group), zero dense columns, a single column / single row, a partition
    wider than the matrix."""
    z = rb.CsrMatrix(5, 7, np.zeros(6, np.int64), np.zeros(0, np.int64), np.zeros(0))
    q = rb.ColumnPartition.uniform(7, 3)
    g = rb.block_1sa(z, q, rb.MergePolicy(tau=0.5))
    assert g.n_groups == 1 and list(g.groups[0].rows) == [0, 1, 2, 3, 4]  # empty rows group together
    V = rb.vbr_from_grouping(z, g, q)
    assert V.n_stored_blocks == 0 and V.stored_area == 0
    for prec in ("bf16", "fp32"):
        C = rb.spmm_vbr(V, rb.DenseMatrix.from_array(np.ones((7, 4))), precision=prec).data
        assert C.shape == (5, 4) and np.all(C == 0.0)
        assert rb.spmm_vbr(V, rb.DenseMatrix.from_array(np.ones((7, 0))), precision=prec).data.shape == (5, 0)
        assert np.all(rb.spmm_csr(z, rb.DenseMatrix.from_array(np.ones((7, 3))), precision=prec).data == 0.0)
    one = rb.CsrMatrix(1, 1, np.array([0, 1]), np.array([0]), np.array([0.5]))
    q1 = rb.ColumnPartition.uniform(1, 64)  # partition wider than the matrix: one ragged segment
    V1 = rb.vbr_from_grouping(one, rb.block_1sa(one, q1, rb.MergePolicy(tau=0.9)), q1)
    for prec in ("bf16", "fp32"):
        C = rb.spmm_vbr(V1, rb.DenseMatrix.from_array(np.array([[2.0, -4.0, 8.0]])), precision=prec).data
        assert np.array_equal(C, np.array([[1.0, -2.0, 4.0]]))


# ------------------------------------------------------------------ 2:4 sparse tensor-core path


@pytest.mark.parametrize("density,N,delta", [(0.01, 300, 64), (0.3, 256, 64), (0.1, 520, 128), (0.5, 64, 192)])
def test_spmm_sparse24_tall_matches_product(density, N, delta):
    """Tall block rows on tcgen05.mma.sp: the compressed 2:4 tiles + TMEM metadata + the residual
    pass (groups with more than two nonzeros) reproduce A·B within the bf16 bound; run-to-run
    bit-identical; dense-tile path agrees to the same bound."""
    from paper_2202_05868_b200.device import DeviceCsr, DeviceVbr
    from paper_2202_05868_b200.types import csr_from_coo

    rng = np.random.default_rng(int(density * 1000) + N)
    heights = [300, 257, 520]
    n_cols = 3000
    rows, cols, r0 = [], [], 0
    for h in heights:
        k = int(density * h * n_cols)
        rows.append(r0 + rng.integers(0, h, k))
        cols.append(rng.integers(0, n_cols, k))
        r0 += h
    keys = np.unique(np.concatenate(rows) * n_cols + np.concatenate(cols))
    vals = rounded(rng.uniform(0.1, 1.0, len(keys)), torch.bfloat16) * rng.choice([-1.0, 1.0], len(keys))
    A = csr_from_coo(r0, n_cols, keys // n_cols, keys % n_cols, vals)
    perm = torch.from_numpy(rng.permutation(r0)).cuda()
    rp = torch.tensor(np.concatenate([[0], np.cumsum(heights)]), device="cuda")
    q = rb.ColumnPartition.uniform(n_cols, delta)
    dv = DeviceVbr.build(DeviceCsr.from_host(A, "cuda"), q, perm, rp, dtypes=("bf16",))
    sp = dv.sparse24("bf16")
    if density >= 0.3:
        assert sp.n_residuals > 0
    Bh = rounded(rng.uniform(-1, 1, (n_cols, N)), torch.bfloat16)
    ld = (N + 7) // 8 * 8
    Bd = torch.zeros((n_cols, ld), dtype=torch.bfloat16, device="cuda")[:, :N]
    Bd.copy_(torch.from_numpy(Bh))
    C1 = dv.spmm(Bd, sparse24=True)
    C2 = dv.spmm(Bd, sparse24=True)
    Cd = dv.spmm(Bd, sparse24=False)
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)
    Ad = A.to_dense()
    bound = np.abs(Ad) @ np.abs(Bh)
    assert_close(C1.cpu().numpy().astype(np.float64), Ad @ Bh, bound, 1e-4, "sparse24")
    assert_close(Cd.cpu().numpy().astype(np.float64), Ad @ Bh, bound, 1e-4, "dense")


@pytest.mark.parametrize("precision,world", [("bf16", 2), ("bf16", 3), ("bf16", 8), ("fp32", 3)])
def test_spmm_shard_plans_cover_rows_and_match_full(precision, world):
    """bench.py --gpus W runs shard k of W on rank k (rb_spmm_plan_create(shard, n_shards)).  Running
    every shard's plan on one device into one C must write every row (NaN-initialised C) and match
    the single-plan product within fp32 reassociation (tall tails are split differently per shard)."""
    from paper_2202_05868_b200 import _lib as L
    from paper_2202_05868_b200.device import DeviceCsr, DeviceVbr

    rng = np.random.default_rng(31 + world)
    heights = [1, 3, 6, 20, 64, 90, 130, 300, 1, 2, 517] * 2  # skinny, short and tall block rows
    A, perm, rp = _grouped_matrix(rng, heights, 1536, 64, 0.02)
    q = rb.ColumnPartition.uniform(1536, 64)
    dt = L.TORCH_DTYPE[L.PRECISION[precision]]
    N = 384
    Bh = rounded(rng.uniform(-1, 1, (1536, N)), dt if dt != torch.float32 else torch.bfloat16)
    Bd = torch.from_numpy(Bh).to(dt).cuda()
    dv = DeviceVbr.build(DeviceCsr.from_host(A, "cuda"), q, perm, rp, dtypes=(precision,))
    full = dv.spmm(Bd, precision=precision)
    C = torch.full_like(full, float("nan"))
    for k in range(world):
        dv.spmm(Bd, out=C, precision=precision, shard=k, n_shards=world)
    torch.cuda.synchronize()
    assert not torch.isnan(C).any(), "a row was not written by any shard"
    err = (C.double() - full.double()).abs().max().item()
    assert err <= 1e-5 * max(1.0, full.abs().max().item())


@pytest.mark.parametrize("precision,world", [("bf16", 4), ("bf16", 8), ("fp32", 8)])
def test_spmm_shard_plans_split_hub_rows(precision, world):
    """Plans with 4+ shards cut skinny block rows into 128-block (4 ranks) / 64-block (8 ranks) parts
    reduced in part order by the last-arriving part.  Skinny rows here hold ~200 blocks (19,200
    columns, Δ=64), so every shard splits them; all rows written, equal to the single plan."""
    from paper_2202_05868_b200 import _lib as L
    from paper_2202_05868_b200.device import DeviceCsr, DeviceVbr

    rng = np.random.default_rng(77 + world)
    heights = [1, 2, 4, 1, 3, 1, 1, 2, 4, 1] * 3
    n_cols = 64 * 300
    A, perm, rp = _grouped_matrix(rng, heights, n_cols, 64, 0.02)
    q = rb.ColumnPartition.uniform(n_cols, 64)
    dt = L.TORCH_DTYPE[L.PRECISION[precision]]
    N = 128
    Bh = rounded(rng.uniform(-1, 1, (n_cols, N)), dt if dt != torch.float32 else torch.bfloat16)
    Bd = torch.from_numpy(Bh).to(dt).cuda()
    dv = DeviceVbr.build(DeviceCsr.from_host(A, "cuda"), q, perm, rp, dtypes=(precision,))
    _, bp, _ = dv.host_structure()
    assert np.diff(bp).max() > 128  # hub rows that the 4/8-rank part sizes cut
    full = dv.spmm(Bd, precision=precision)
    C = torch.full_like(full, float("nan"))
    for k in range(world):
        dv.spmm(Bd, out=C, precision=precision, shard=k, n_shards=world)
    torch.cuda.synchronize()
    assert not torch.isnan(C).any(), "a row was not written by any shard"
    err = (C.double() - full.double()).abs().max().item()
    assert err <= 1e-5 * max(1.0, full.abs().max().item())
    ref = torch.from_numpy(A.to_dense() @ Bh).cuda()
    assert ((C.double() - ref).abs().max() <= 1e-4 * max(1.0, ref.abs().max().item())).item()


def test_spmm_fp64_golden_small(golden_small):
    """fp64 path (float64 CUDA-core kernel over the dense payloads): C within 1e-12 (scaled by |A|·|B|)
    of the reference's float64 C on every golden case with B; empty rows exactly 0."""
    n = 0
    for name, case in golden_small.items():
        B = golden_b(case)
        if B is None or "C" not in case:
            continue
        A, q = csr_of(case), part_of(case)
        V = rb.vbr_from_grouping(A, rb.block_1sa(A, q, policy_of(case), bool(case["use_compression"])), q)
        C = rb.spmm_vbr(V, rb.DenseMatrix.from_array(B), precision="fp64").data
        ref = case["C"]
        bound = np.abs(dense_of(case)) @ np.abs(B)  # mixed-sign cases cancel: scale by |A|·|B|
        assert_close(C, ref, bound, 1e-12, name)
        empty = np.diff(case["row_ptr"]) == 0
        assert np.all(C[empty] == 0.0), name
        n += 1
    assert n > 100


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_spmm_fp64_propagates_nonfinite_like_the_reference(bad):
    """With precision="fp64" a NaN / Inf in B propagates exactly as the reference's dense-payload
    product does (0 * NaN = NaN inside a stored block's segment, 0 * Inf = NaN, Inf of both signs
    -> NaN), checked against the oracle's numpy restatement of multiply.py:72-97."""
    import oracle

    case = load_golden("cfg1_full")
    A, q = csr_of(case), part_of(case)
    V = rb.vbr_from_grouping(A, rb.block_1sa(A, q, policy_of(case), True), q)
    B = np.random.default_rng(3).random((A.n_cols, 16))
    B[17, 5] = bad
    B[900, 3] = -bad if not np.isnan(bad) else bad
    C = rb.spmm_vbr(V, rb.DenseMatrix.from_array(B), precision="fp64").data
    bp, bc = oracle.vbr_blocks(case["row_ptr"], case["col_idx"], case["boundaries"], case["row_perm"],
                               case["row_partition"])
    pay = oracle.vbr_payloads(case["row_ptr"], case["col_idx"], case["values"], case["boundaries"],
                              case["row_perm"], case["row_partition"], bp, bc)
    ref = oracle.spmm_vbr_np(pay, case["row_perm"], case["row_partition"], case["boundaries"], B)
    assert np.array_equal(np.isnan(C), np.isnan(ref))
    assert np.array_equal(np.isposinf(C), np.isposinf(ref)) and np.array_equal(np.isneginf(C), np.isneginf(ref))
    fin = np.isfinite(ref)
    assert np.isnan(ref).any() and np.allclose(C[fin], ref[fin], rtol=1e-12, atol=0)

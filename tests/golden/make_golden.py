"""Generate golden fixtures by running the REFERENCE implementation (rowblock v0.1.0).

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/golden_*.npz``.  Each case holds the input CSR, the
column partition, the merge policy, the reference's grouping / VBR structure
(block_1sa, blocking.py:283; vbr_from_grouping, vbr.py:88) and, for the small
cases, B and the reference's C = spmm_vbr(V, B) (multiply.py:72).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import rowblock as rb  # noqa: E402
from rowblock.matrix import _csr_from_coo  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def random_csr(rng, n_rows, n_cols, density, positive=True):
    # same construction as the reference's tests/conftest.py:7-16
    nnz = min(n_rows * n_cols, max(1, round(density * n_rows * n_cols)))
    keys = rng.choice(n_rows * n_cols, size=nnz, replace=False)
    vals = rng.uniform(0.1, 1.0, size=nnz)
    if not positive:
        vals *= rng.choice([-1.0, 1.0], size=nnz)
    return _csr_from_coo(n_rows, n_cols, keys // n_cols, keys % n_cols, vals, sum_duplicates=False)


def record(name, A, q, policy, use_compression=True, B=None, store_c=True, b_seed=None):
    g = rb.block_1sa(A, q, policy, use_compression=use_compression)
    rb.check_grouping(A, q, g)
    V = rb.vbr_from_grouping(A, g, q)
    d = dict(
        n_rows=A.n_rows, n_cols=A.n_cols, row_ptr=A.row_ptr, col_idx=A.col_idx, values=A.values,
        boundaries=q.boundaries, tau=policy.tau, cosine=int(policy.similarity == "cosine"),
        bounded=int(policy.bounded), pattern_update=int(policy.pattern_update),
        use_compression=int(use_compression),
        group_of=g.group_of,
        group_ptr=np.concatenate([[0], np.cumsum(g.heights())]).astype(np.int64),
        row_perm=V.row_perm, row_partition=V.row_partition,
        seed_size=np.array([grp.seed_size for grp in g.groups], np.int64),
        pattern_ptr=np.concatenate([[0], np.cumsum([len(grp.pattern) for grp in g.groups])]).astype(np.int64),
        pattern_idx=(np.concatenate([grp.pattern for grp in g.groups]) if g.n_groups else np.zeros(0)).astype(np.int64),
        blk_ptr=np.concatenate([[0], np.cumsum([len(br) for br in V.block_rows])]).astype(np.int64),
        blk_col=np.array([b.bcol for br in V.block_rows for b in br], np.int64),
        stored_area=V.stored_area,
    )
    if B is not None:
        C = rb.spmm_vbr(V, rb.DenseMatrix.from_array(B)).data
        if b_seed is None:
            d["B"] = B
        else:  # regenerate with np.random.default_rng(b_seed).random(B_shape)
            d["B_seed"] = b_seed
            d["B_shape"] = np.array(B.shape)
        if store_c:
            d["C"] = C
        # size-independent checksums of C (always stored)
        r = np.random.default_rng(7).standard_normal(B.shape[1])
        d["C_dot_r"] = C @ r
        d["C_rowsum"] = C.sum(axis=1)
    return name, d


def hand_matrix():
    return rb.csr_from_triplets(4, 6, [(0, 0, 1.0), (0, 1, 1.0), (1, 3, 1.0), (2, 2, 1.0), (3, 4, 1.0),
                                       (3, 5, 1.0)])


def kat_cases():
    cases = []
    P = rb.MergePolicy
    Q = rb.ColumnPartition.uniform
    A = hand_matrix()
    for bounded in (True, False):
        for comp in (True, False):
            cases.append(record(f"kat_hand_b{int(bounded)}_c{int(comp)}", A, Q(6, 3), P(tau=0.5, bounded=bounded),
                                comp, B=np.ones((6, 2))))
    S = rb.csr_from_triplets(4, 4, [(0, 0, 1.0), (1, 2, 1.0), (2, 0, 1.0), (2, 2, 1.0), (3, 3, 1.0)])
    cases.append(record("kat_single_pass_upd", S, Q(4, 2), P(tau=0.5, bounded=False, pattern_update=True), False))
    cases.append(record("kat_single_pass_noupd", S, Q(4, 2), P(tau=0.5, bounded=False, pattern_update=False), False))
    cases.append(record("kat_single_pass_comp", S, Q(4, 2), P(tau=0.5, bounded=False, pattern_update=True), True))
    E = rb.csr_from_triplets(4, 4, [(1, 0, 1.0), (3, 0, 1.0)])
    cases.append(record("kat_empty_rows", E, Q(4, 2), P(tau=0.5), True, B=np.arange(8.0).reshape(4, 2)))
    cases.append(record("kat_empty_rows_nocomp", E, Q(4, 2), P(tau=0.5), False))
    I5 = rb.csr_from_triplets(5, 4, [(i, c, 1.0) for i in range(5) for c in (1, 3)])
    cases.append(record("kat_identical", I5, Q(4, 1), P(tau=0.9), True))
    D4 = rb.csr_from_triplets(4, 4, [(i, i, 1.0) for i in range(4)])
    cases.append(record("kat_tau1_distinct", D4, Q(4, 1), P(tau=1.0), True, B=np.eye(4)))
    rng = np.random.default_rng(20240917)
    cases.append(record("kat_tau0_unbounded", random_csr(rng, 12, 16, 0.2), Q(16, 4), P(tau=0.0, bounded=False), True))
    Z = rb.csr_from_triplets(3, 3, [])
    cases.append(record("kat_all_empty", Z, Q(3, 2), P(tau=0.5), True, B=np.ones((3, 2))))
    cases.append(record("kat_pathological_b", rb.pathological_matrix(256), Q(rb.pathological_matrix(256).n_cols, 1),
                        P(tau=0.5, bounded=True), True))
    cases.append(record("kat_pathological_u", rb.pathological_matrix(256), Q(rb.pathological_matrix(256).n_cols, 1),
                        P(tau=0.5, bounded=False), True))
    return cases


def random_cases(n_cases=120):
    cases = []
    for k in range(n_cases):
        rng = np.random.default_rng(50_000 + k)
        n = int(rng.integers(1, 200))
        m = int(rng.integers(1, 200))
        dens = float(rng.choice([0.005, 0.02, 0.05, 0.1, 0.25, 0.5]))
        A = random_csr(rng, n, m, dens, positive=bool(rng.integers(2)))
        # sprinkle empty rows
        if rng.random() < 0.3 and n > 2:
            keep = rng.random(n) < 0.7
            rows = np.repeat(np.arange(n), np.diff(A.row_ptr))
            mask = keep[rows]
            A = _csr_from_coo(n, m, rows[mask], A.col_idx[mask], A.values[mask], sum_duplicates=False)
        dw = int(rng.choice([1, 2, 3, 4, 5, 7, 8, 16, 32, 64, 100]))
        q = rb.ColumnPartition.uniform(m, dw)
        policy = rb.MergePolicy(similarity=str(rng.choice(["jaccard", "cosine"])),
                                tau=float(rng.choice([0.0, 0.1, 0.2, 0.3, 0.5, 0.7, 0.8, 0.9, 1.0])),
                                bounded=bool(rng.integers(2)), pattern_update=bool(rng.integers(2)))
        comp = bool(rng.integers(2))
        N = int(rng.integers(1, 40))
        B = rng.random((m, N))
        cases.append(record(f"rand_{k:03d}", A, q, policy, comp, B=B))
    return cases


def nonuniform_cases():
    cases = []
    for k in range(12):
        rng = np.random.default_rng(60_000 + k)
        n, m = int(rng.integers(10, 120)), int(rng.integers(10, 150))
        A = random_csr(rng, n, m, float(rng.choice([0.03, 0.1, 0.3])))
        cuts = np.unique(rng.integers(1, m, size=int(rng.integers(1, max(2, m // 3)))))
        q = rb.ColumnPartition(m, np.concatenate([[0], cuts, [m]]))
        pol = rb.MergePolicy(tau=float(rng.choice([0.3, 0.5, 0.7])), bounded=bool(rng.integers(2)))
        cases.append(record(f"nonuni_{k:02d}", A, q, pol, True, B=rng.random((m, 9))))
    return cases


def rmat_cases():
    """Config 3 flavour (R-MAT, rows scrambled, Δ=32) with B, so the skinny SpMM path is checked
    against spmm_vbr (multiply.py:72-97) on power-law input: 2^12 at τ ∈ {0.3, 0.9} (N=64) and
    2^16 at τ=0.7 (N=128, config 3's N; C checksums only)."""
    cases = []
    R = rb.gen_rmat(rb.RmatSpec(12, 16, seed=3))
    Rs, _ = rb.scramble(R, 33)
    for tau in (0.3, 0.9):
        cases.append(record(f"rmat12_t{int(tau * 10)}", Rs, rb.ColumnPartition.uniform(R.n_cols, 32),
                            rb.MergePolicy(tau=tau), True, B=np.random.default_rng(34).random((R.n_cols, 64)),
                            store_c=False, b_seed=34))
    R = rb.gen_rmat(rb.RmatSpec(16, 16, seed=3))
    Rs, _ = rb.scramble(R, 36)
    cases.append(record("rmat16_t7", Rs, rb.ColumnPartition.uniform(R.n_cols, 32), rb.MergePolicy(tau=0.7), True,
                        B=np.random.default_rng(37).random((R.n_cols, 128)), store_c=False, b_seed=37))
    return cases


def medium_cases():
    """Scaled versions of the BASELINE configs (structure + C checksums)."""
    cases = []
    # config 1 exactly: 2048^2, 1% uniform (gen_blocked(2048,2048,1,0.01,1.0)), Δ=64, τ=0.7, N=256
    A = rb.gen_blocked(rb.BlockedMatrixSpec(2048, 2048, 1, 0.01, 1.0, seed=1))
    rng = np.random.default_rng(11)
    vals = rng.uniform(0.1, 1.0, A.nnz)
    A = rb.CsrMatrix(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, vals)
    cases.append(record("cfg1_full", A, rb.ColumnPartition.uniform(2048, 64), rb.MergePolicy(tau=0.7), True,
                        B=np.random.default_rng(12).random((2048, 256)), store_c=False, b_seed=12))
    # config 5 at 1/32 linear scale: 8192^2, 64^2 blocks θ=1%, ρ=1, rows scrambled, Δ=64
    A = rb.gen_blocked(rb.BlockedMatrixSpec(8192, 8192, 64, 0.01, 1.0, seed=5))
    S, _ = rb.scramble(A, 55)
    cases.append(record("cfg5_s32", S, rb.ColumnPartition.uniform(8192, 64), rb.MergePolicy(tau=0.7), True,
                        B=np.random.default_rng(56).random((8192, 64)), store_c=False, b_seed=56))
    # config 4 at 1/8 rows x 1/4 cols: 512x4096, 10% uniform, Δ=128
    rng = np.random.default_rng(44)
    A = random_csr(rng, 512, 4096, 0.1)
    cases.append(record("cfg4_s8", A, rb.ColumnPartition.uniform(4096, 128), rb.MergePolicy(tau=0.7), True,
                        B=np.random.default_rng(45).random((4096, 128)), store_c=False, b_seed=45))
    cases += rmat_cases()
    # hidden blocks + noise, rows scrambled only (config 2b flavour) at 2048^2
    A = rb.gen_blocked(rb.BlockedMatrixSpec(2048, 2048, 64, 0.05, 1.0, seed=2))
    S, _ = rb.scramble(A, 22)
    cases.append(record("cfg2b_s16", S, rb.ColumnPartition.uniform(2048, 64), rb.MergePolicy(tau=0.7), True))
    return cases


def main():
    if "--rmat" in sys.argv:  # regenerate only the R-MAT cases
        for n, d in rmat_cases():
            np.savez_compressed(os.path.join(OUT, f"golden_{n}.npz"), **{k: np.asarray(v) for k, v in d.items()})
            print("wrote", n)
        return
    allc = kat_cases() + random_cases() + nonuniform_cases() + medium_cases()
    small = {n: d for n, d in allc if not n.startswith(("cfg", "rmat"))}
    np.savez_compressed(os.path.join(OUT, "golden_small.npz"),
                        **{f"{n}__{k}": np.asarray(v) for n, d in small.items() for k, v in d.items()})
    for n, d in allc:
        if n.startswith(("cfg", "rmat")):
            np.savez_compressed(os.path.join(OUT, f"golden_{n}.npz"), **{k: np.asarray(v) for k, v in d.items()})
    print(f"wrote {len(allc)} cases")


if __name__ == "__main__":
    main()

"""TEST INFRASTRUCTURE ONLY — CPU oracle for the rowblock hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package, and only
as the checker or the timed CPU baseline.  The product package
``paper_2202_05868_b200`` never imports it.

Parity is pinned: ``tests/test_oracle.py`` checks this restatement against
golden vectors produced by running the reference itself
(``tests/golden/make_golden.py`` → ``tests/golden/*.npz``) and against the
reference's own known-answer tests.

Contents
--------
* ``block_1sa_arrays`` / ``quotient`` / ``vbr_blocks``: ctypes bindings to
  ``rowblock_oracle.c`` (C restatement of blocking.py:118-306, vbr.py:88-125).
* ``vbr_payloads``: the float64 block payloads (``orc_vbr_scatter``, vbr.py:113-123).
* ``spmm_vbr_np`` / ``spmm_csr_np``: numpy restatements of multiply.py:51-97
  (float64, per-block dgemm, the same ThreadPool chunking over block rows).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liborc.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C restatement (gcc -O2, no -ffast-math: IEEE compares must match numpy)."""
    src = os.path.join(_HERE, "rowblock_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        lib.orc_quotient.argtypes = [I, P, P, P, I, P, P]
        lib.orc_block_1sa.argtypes = [I, P, P, P, I, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, P, P, P, P, P, P, P]
        lib.orc_vbr_blocks.argtypes = [I, P, P, P, I, P, P, I, P, P]
        lib.orc_vbr_scatter.argtypes = [I, P, P, P, P, P, P, I, P, P, P, P]
        lib.orc_block_1sa_pruned.argtypes = [I, P, P, P, I, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_int, P, P, P, P, P, P, P, P]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _c64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def quotient(row_ptr, col_idx, boundaries):
    """(bits uint64[n, W], sizes int64[n]) — blocking.py:118-136."""
    row_ptr, col_idx, b = _c64(row_ptr), _c64(col_idx), _c64(boundaries)
    n = len(row_ptr) - 1
    n_seg = len(b) - 1
    W = max(1, (n_seg + 63) // 64)
    bits = np.zeros((n, W), dtype=np.uint64)
    sizes = np.zeros(n, dtype=np.int64)
    _load().orc_quotient(n, _ptr(row_ptr), _ptr(col_idx), _ptr(b), n_seg, _ptr(bits), _ptr(sizes))
    return bits, sizes


def block_1sa_arrays(row_ptr, col_idx, boundaries, tau=0.5, similarity="jaccard", bounded=True,
                     pattern_update=True, use_compression=True, pruned=False) -> dict:
    """Array form of block_1sa (blocking.py:283-306).

    Returns dict(group_of, row_perm, group_ptr, seed_size, pattern_ptr, pattern_idx, n_groups).
    """
    row_ptr, col_idx, b = _c64(row_ptr), _c64(col_idx), _c64(boundaries)
    n = len(row_ptr) - 1
    nnz = int(row_ptr[-1]) if n >= 0 else 0
    n_seg = len(b) - 1
    out = dict(
        group_of=np.zeros(max(n, 1), np.int64), row_perm=np.zeros(max(n, 1), np.int64),
        group_ptr=np.zeros(n + 1, np.int64), seed_size=np.zeros(max(n, 1), np.int64),
        pattern_ptr=np.zeros(n + 1, np.int64), pattern_idx=np.zeros(max(nnz, 1), np.int64),
    )
    H = np.zeros(1, np.int64)
    args = (n, _ptr(row_ptr), _ptr(col_idx), _ptr(b), n_seg, float(tau), int(similarity == "cosine"),
            int(bool(bounded)), int(bool(pattern_update)), int(bool(use_compression)), _ptr(out["group_of"]),
            _ptr(out["row_perm"]), _ptr(out["group_ptr"]), _ptr(out["seed_size"]), _ptr(out["pattern_ptr"]),
            _ptr(out["pattern_idx"]), _ptr(H))
    if pruned:
        stats = np.zeros(3, np.int64)
        rc = _load().orc_block_1sa_pruned(*args, _ptr(stats))
        out["stats"] = dict(rounds=int(stats[0]), postings_visited=int(stats[1]), candidates=int(stats[2]))
    else:
        rc = _load().orc_block_1sa(*args)
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    h = int(H[0])
    out["n_groups"] = h
    out["group_of"] = out["group_of"][:n]
    out["row_perm"] = out["row_perm"][:n]
    out["group_ptr"] = out["group_ptr"][: h + 1]
    out["seed_size"] = out["seed_size"][:h]
    out["pattern_ptr"] = out["pattern_ptr"][: h + 1]
    out["pattern_idx"] = out["pattern_idx"][: int(out["pattern_ptr"][-1])]
    return out


def vbr_blocks(row_ptr, col_idx, boundaries, row_perm, row_partition):
    """(blk_ptr int64[H+1], blk_col int64[nb]) — vbr.py:106-112."""
    row_ptr, col_idx, b = _c64(row_ptr), _c64(col_idx), _c64(boundaries)
    row_perm, row_partition = _c64(row_perm), _c64(row_partition)
    n = len(row_ptr) - 1
    H = len(row_partition) - 1
    nnz = int(row_ptr[-1])
    blk_ptr = np.zeros(H + 1, np.int64)
    blk_col = np.zeros(max(nnz, 1), np.int64)
    rc = _load().orc_vbr_blocks(n, _ptr(row_ptr), _ptr(col_idx), _ptr(b), len(b) - 1, _ptr(row_perm),
                                _ptr(row_partition), H, _ptr(blk_ptr), _ptr(blk_col))
    if rc != 0:
        raise ValueError("oracle: bad row_perm")
    return blk_ptr, blk_col[: int(blk_ptr[-1])]


# ---------------------------------------------------------------------------
# SpMM restatements (multiply.py:43-97), float64


def _chunks(n: int, parts: int):
    # multiply.py:43-48
    if n == 0:
        return []
    parts = max(1, min(parts, n))
    step = (n + parts - 1) // parts
    return [(lo, min(lo + step, n)) for lo in range(0, n, step)]


def vbr_payloads(row_ptr, col_idx, values, boundaries, row_perm, row_partition, blk_ptr, blk_col):
    """Dense float64 payload per stored block (vbr.py:113-123), scattered by ``orc_vbr_scatter``.

    Returns a list (per block row g) of lists of (bcol, payload[h_g, w_bcol]) with bcols ascending;
    every payload is a view into one flat float64 buffer.
    """
    row_ptr, col_idx, b = _c64(row_ptr), _c64(col_idx), _c64(boundaries)
    values = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    rp, bp, bc = _c64(row_partition), _c64(blk_ptr), _c64(blk_col)
    perm = _c64(row_perm)
    n = len(row_ptr) - 1
    H = len(rp) - 1
    widths = np.diff(b)
    heights = np.diff(rp)
    blk_h = np.repeat(heights, np.diff(bp))
    blk_w = widths[bc] if len(bc) else np.zeros(0, np.int64)
    blk_off = np.zeros(len(bc) + 1, np.int64)
    np.cumsum(blk_h * blk_w, out=blk_off[1:])
    flat = np.zeros(max(int(blk_off[-1]), 1), np.float64)
    if len(col_idx):
        rc = _load().orc_vbr_scatter(n, _ptr(row_ptr), _ptr(col_idx), _ptr(values), _ptr(b), _ptr(perm), _ptr(rp), H,
                                     _ptr(bp), _ptr(bc), _ptr(blk_off), _ptr(flat))
        if rc != 0:
            raise ValueError("nonzero outside the stored blocks" if rc == -3 else "oracle: bad row_perm")
    out = []
    for gg in range(H):
        out.append([(int(bc[k]), flat[blk_off[k]:blk_off[k + 1]].reshape(int(blk_h[k]), int(blk_w[k])))
                    for k in range(int(bp[gg]), int(bp[gg + 1]))])
    return out


def spmm_vbr_np(payloads, row_perm, row_partition, boundaries, B: np.ndarray, threads: int = 1,
                block_rows=None, out=None) -> np.ndarray:
    """multiply.py:72-97: per block row, acc = sum over blocks (ascending bcol) of payload @ B panel,
    then C[row_perm[lo:hi]] = acc.  Empty block rows are skipped (their C rows stay exactly 0).
    ``block_rows`` restricts the product to those block rows; ``out`` receives their C rows."""
    n_rows = len(row_perm)
    B = np.asarray(B, dtype=np.float64)
    C = np.zeros((n_rows, B.shape[1])) if out is None else out
    b = _c64(boundaries)
    rp = _c64(row_partition)
    perm = _c64(row_perm)
    todo = list(range(len(rp) - 1)) if block_rows is None else list(block_rows)

    def run(span):
        for gi in range(*span):
            g = todo[gi]
            lo, hi = int(rp[g]), int(rp[g + 1])
            if hi == lo or not payloads[g]:
                continue
            acc = np.zeros((hi - lo, B.shape[1]))
            for s, pay in payloads[g]:
                acc += pay @ B[b[s]:b[s + 1]]
            C[perm[lo:hi]] = acc

    if threads > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(run, _chunks(len(todo), threads)))
    else:
        run((0, len(todo)))
    return C


def spmm_csr_np(row_ptr, col_idx, values, B: np.ndarray) -> np.ndarray:
    """multiply.py:51-69 (single thread): C[i] = values[s:e] @ B[col_idx[s:e]]."""
    row_ptr, col_idx = _c64(row_ptr), _c64(col_idx)
    values = np.asarray(values, dtype=np.float64)
    n = len(row_ptr) - 1
    B = np.asarray(B, dtype=np.float64)
    C = np.zeros((n, B.shape[1]))
    for i in range(n):
        s, e = row_ptr[i], row_ptr[i + 1]
        if e > s:
            C[i] = values[s:e] @ B[col_idx[s:e]]
    return C


def group_stats_np(row_ptr, col_idx, boundaries, row_perm, group_ptr, pattern_ptr, pattern_idx, tau):
    """Restatement of blocking_stats (metrics.py:59-95) and verify_density_bound (metrics.py:178-216)
    on grouping arrays: per group stored columns, element nnz, quotient nnz (popcount of the
    quotient bits, blocking.py:118-136) and the exact Fraction verdicts; plus the totals."""
    from fractions import Fraction

    rp = np.asarray(row_ptr, np.int64)
    b = np.asarray(boundaries, np.int64)
    widths = np.diff(b)
    max_w = int(widths.max()) if len(widths) else 1
    _, qsizes = quotient(rp, col_idx, b)
    row_nnz = np.diff(rp)
    f_tau = Fraction(float(tau))
    eb, qb = f_tau / (2 * max_w), f_tau / 2
    gp, pp = np.asarray(group_ptr, np.int64), np.asarray(pattern_ptr, np.int64)
    perm, pats = np.asarray(row_perm, np.int64), np.asarray(pattern_idx, np.int64)
    H = len(gp) - 1
    out = {k: np.zeros(H, np.int64) for k in ("stored_cols", "element_nnz", "quotient_nnz")}
    out["element_ok"] = np.ones(H, bool)
    out["quotient_ok"] = np.ones(H, bool)
    area = blocks = hsum = 0
    for g in range(H):
        rows = perm[gp[g]:gp[g + 1]]
        pat = pats[pp[g]:pp[g + 1]]
        h, lam = len(rows), len(pat)
        sc = int(widths[pat].sum()) if lam else 0
        ke, kq = int(row_nnz[rows].sum()), int(np.asarray(qsizes)[rows].sum())
        out["stored_cols"][g], out["element_nnz"][g], out["quotient_nnz"][g] = sc, ke, kq
        area += h * sc
        blocks += lam
        hsum += h * lam
        if lam:
            out["element_ok"][g] = Fraction(ke, h * sc) >= eb
            out["quotient_ok"][g] = Fraction(kq, h * lam) >= qb
    out.update(stored_area=area, n_blocks=blocks, height_sum=hsum, nnz=int(rp[-1]), n_groups=H,
               element_bound=float(eb), quotient_bound=float(qb))
    return out

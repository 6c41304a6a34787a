"""MatrixMarket coordinate files — drop-in for rowblock.mtxio (mtxio.py:1-119), vectorised.

Accepted: ``coordinate`` layout; ``real`` / ``integer`` / ``pattern`` fields; ``general`` /
``symmetric`` storage.  Canonicalisation follows the reference: pattern entries are 1.0,
symmetric storage is mirrored, duplicates are summed in file order, zeros are dropped.  Errors are
``MatrixMarketError`` (a ValueError) with the reference's messages and 1-based line numbers.

The entry block is parsed by one structured ``np.loadtxt`` call (integers as integers, values with a
correctly rounded decimal conversion, as ``float()``); only a file that parse rejects is walked line
by line, to name the offending line.  ``read_matrix_market_device`` lands the CSR in HBM.
"""

from __future__ import annotations

import io

import numpy as np

from .types import CsrMatrix, csr_from_coo

__all__ = ["MatrixMarketError", "read_matrix_market", "read_matrix_market_device", "write_matrix_market"]

_ALLOWED = {"layout": ("coordinate",), "field": ("real", "integer", "pattern"), "symmetry": ("general", "symmetric")}


class MatrixMarketError(ValueError):
    """A malformed or unsupported file; ``path`` and ``lineno`` locate the problem."""

    def __init__(self, path, lineno, message):
        super().__init__(f"{path}:{lineno}: {message}")
        self.path, self.lineno = str(path), lineno


def _banner(path, line: str):
    if not line.lower().startswith("%%matrixmarket"):
        raise MatrixMarketError(path, 1, "missing %%MatrixMarket header")
    words = line.strip().split()
    if len(words) != 5 or words[1].lower() != "matrix":
        raise MatrixMarketError(path, 1, f"malformed header: {line.strip()!r}")
    layout, fld, sym = (w.lower() for w in words[2:])
    for kind, value in (("layout", layout), ("field", fld), ("symmetry", sym)):
        if value not in _ALLOWED[kind]:
            extra = " (only coordinate)" if kind == "layout" else ""
            raise MatrixMarketError(path, 1, f"unsupported {kind} {value!r}{extra}")
    return fld, sym


def _content(lines, first_lineno):
    """(lineno, stripped line) for every non-blank, non-comment line."""
    for k, raw in enumerate(lines):
        text = raw.strip()
        if text and not text.startswith("%"):
            yield first_lineno + k, text


def _diagnose(path, lines, first_lineno, shape, want):
    """Walk the entries the reference's way to report the first bad line (mtxio.py:69-92)."""
    n_rows, n_cols, n_entries = shape
    seen, last = 0, first_lineno - 1
    for lineno, text in _content(lines, first_lineno):
        last = lineno
        toks = text.split()
        if len(toks) != want:
            raise MatrixMarketError(path, lineno, f"expected {want} fields, got {len(toks)}")
        if seen >= n_entries:
            raise MatrixMarketError(path, lineno, "more entries than declared")
        try:
            i, j = int(toks[0]), int(toks[1])
            if want == 3:
                float(toks[2])
        except ValueError:
            raise MatrixMarketError(path, lineno, f"bad entry {text!r}") from None
        if not (1 <= i <= n_rows and 1 <= j <= n_cols):
            raise MatrixMarketError(path, lineno, f"index ({i}, {j}) out of range")
        seen += 1
    last = max(last, first_lineno - 1 + len(lines))
    if seen != n_entries:
        raise MatrixMarketError(path, last, f"declared {n_entries} entries, found {seen}")
    raise MatrixMarketError(path, last, "malformed entry block")


def read_matrix_market(path) -> CsrMatrix:
    """Canonical CsrMatrix from a MatrixMarket coordinate file (mtxio.py:30-107)."""
    with open(path, "r", encoding="ascii", errors="replace") as fh:
        text = fh.read()
    lines = text.split("\n")
    if text.endswith("\n"):
        lines.pop()
    fld, sym = _banner(path, lines[0] if lines else "")
    shape, body_at = None, len(lines)
    for lineno, line in _content(lines[1:], 2):
        toks = line.split()
        if len(toks) != 3:
            raise MatrixMarketError(path, lineno, "size line must be 'rows cols nnz'")
        try:
            shape = tuple(int(t) for t in toks)
        except ValueError:
            raise MatrixMarketError(path, lineno, f"bad size line {line!r}") from None
        body_at = lineno  # entries start on the next line
        break
    if shape is None:
        raise MatrixMarketError(path, len(lines), "missing size line")
    if min(shape) < 0:
        raise MatrixMarketError(path, body_at, "negative size")
    n_rows, n_cols, n_entries = shape
    body = lines[body_at:]
    want = 2 if fld == "pattern" else 3
    columns = [("i", np.int64), ("j", np.int64)] + ([("v", np.float64)] if want == 3 else [])
    entries = [t for _, t in _content(body, body_at + 1)]
    try:
        if len(entries) != n_entries:
            raise ValueError("entry count")
        rec = (np.loadtxt(io.StringIO("\n".join(entries)), dtype=np.dtype(columns), ndmin=1) if n_entries
               else np.zeros(0, dtype=np.dtype(columns)))
        r0, c0 = rec["i"] - 1, rec["j"] - 1
        if n_entries and not (0 <= r0.min() and r0.max() < n_rows and 0 <= c0.min() and c0.max() < n_cols):
            raise ValueError("index range")
    except ValueError:
        _diagnose(path, body, body_at + 1, shape, want)
    vals = rec["v"].astype(np.float64) if want == 3 else np.ones(n_entries)
    if sym == "symmetric":
        mirror = r0 != c0
        r0, c0 = np.r_[r0, c0[mirror]], np.r_[c0, r0[mirror]]
        vals = np.r_[vals, vals[mirror]]
    return csr_from_coo(n_rows, n_cols, r0, c0, vals, sum_duplicates=True)


def read_matrix_market_device(path, device=None):
    """read_matrix_market straight into HBM (DeviceCsr: int64 row_ptr / col_idx, float64 values)."""
    from .device import DeviceCsr

    A = read_matrix_market(path)
    dA = DeviceCsr.from_host(A, device)
    dA.source = A
    return dA


def write_matrix_market(path, A: CsrMatrix, comment: str | None = None) -> None:
    """``coordinate real general``, 1-based, ``%.17g`` values — byte-identical to the reference's
    writer (mtxio.py:110-119)."""
    head = ["%%MatrixMarket matrix coordinate real general"]
    head += [f"% {ln}" for ln in (comment.splitlines() if comment else [])]
    head.append(f"{A.n_rows} {A.n_cols} {A.nnz}")
    rows1 = np.repeat(np.arange(1, A.n_rows + 1, dtype=np.int64), A.row_nnz()).tolist()
    body = (f"{i} {j + 1} {v:.17g}" for i, j, v in zip(rows1, A.col_idx.tolist(), A.values.tolist()))
    with open(path, "w", encoding="ascii") as fh:
        fh.write("\n".join(head) + "\n")
        fh.writelines(line + "\n" for line in body)

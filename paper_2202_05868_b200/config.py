"""Process-wide defaults of the drop-in API."""

from __future__ import annotations

import os

_PRECISION = os.environ.get("ROWBLOCK_B200_PRECISION", "bf16")


def default_precision() -> str:
    """Kernel precision used by vbr_from_grouping / spmm_vbr when none is given:
    "bf16" (tcgen05, default), "fp16" (tcgen05), "fp32" (check path) or "fp64" (float64 CUDA-core
    path: the reference's arithmetic, ~1e-15 relative, NaN / Inf of B propagated as multiply.py:89)."""
    return _PRECISION


def set_default_precision(p: str) -> None:
    global _PRECISION
    if p not in ("bf16", "fp16", "fp32", "fp64"):
        raise ValueError(f"unknown precision {p!r}")
    _PRECISION = p


_SPARSE24 = os.environ.get("ROWBLOCK_B200_SPARSE24", "0") not in ("", "0", "false", "no")


def default_sparse24() -> bool:
    """Whether bf16/fp16 SpMM plans run the tall block rows on the 2:4 sparse tensor cores
    (tcgen05.mma.sp over the compressed tiles + residual pass) instead of the dense tiles."""
    return _SPARSE24


def set_default_sparse24(on: bool) -> None:
    global _SPARSE24
    _SPARSE24 = bool(on)


_COMPACT_H = int(os.environ.get("RB_COMPACT_H", "8"))  # all skinny block rows (h <= 4 tensor path, <= 8 fp32)


def compact_h() -> int:
    """Block rows of at most this many rows are multiplied from compact payloads (their nonzeros in
    block-column order, no segment padding) instead of their tiles; 0 = always the tiles."""
    return _COMPACT_H


def set_compact_h(h: int) -> None:
    global _COMPACT_H
    _COMPACT_H = max(0, min(8, int(h)))

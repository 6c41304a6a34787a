"""Process-wide defaults of the drop-in API."""

from __future__ import annotations

import os

_PRECISION = os.environ.get("ROWBLOCK_B200_PRECISION", "bf16")


def default_precision() -> str:
    """Kernel precision used by vbr_from_grouping / spmm_vbr when none is given:
    "bf16" (tcgen05, default), "fp16" (tcgen05) or "fp32" (check path)."""
    return _PRECISION


def set_default_precision(p: str) -> None:
    global _PRECISION
    if p not in ("bf16", "fp16", "fp32"):
        raise ValueError(f"unknown precision {p!r}")
    _PRECISION = p

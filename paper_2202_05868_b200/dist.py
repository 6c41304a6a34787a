"""Block-row sharding of the SpMM across ranks (one process per GPU) — SURVEY.md §8(e).

Each rank owns a contiguous, work-balanced range of PERMUTED rows (whole
block-row M-tiles, ``rb_spmm_shard_range``), so it writes a disjoint set of C
rows with no data-path collective.  B is replicated.  The only collective is the
optional all-gather of C: every rank's rows (in permuted order) are gathered
with ``torch.distributed.all_gather`` (NCCL over NVLink on the GPU
box, gloo in the CPU tests) and un-permuted in place.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L


def shard_range(row_partition, blk_ptr, precision: str, dp: int, shard: int, n_shards: int) -> tuple[int, int]:
    """[row_begin, row_end) of permuted rows owned by ``shard`` (host arrays; no GPU needed)."""
    rp = np.ascontiguousarray(np.asarray(row_partition, np.int32))
    bp = np.ascontiguousarray(np.asarray(blk_ptr, np.int32))
    b, e = ctypes.c_int64(0), ctypes.c_int64(0)
    L.check(L.lib().rb_spmm_shard_range(rp.ctypes.data_as(ctypes.c_void_p), bp.ctypes.data_as(ctypes.c_void_p),
                                        len(rp) - 1, L.PRECISION[precision], int(dp), int(shard), int(n_shards),
                                        ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


def all_ranges(row_partition, blk_ptr, precision: str, dp: int, n_shards: int) -> list[tuple[int, int]]:
    return [shard_range(row_partition, blk_ptr, precision, dp, k, n_shards) for k in range(n_shards)]


def gather_c(C_local: torch.Tensor, row_perm: torch.Tensor, ranges, group=None) -> torch.Tensor:
    """All-gather C.

    ``C_local``: this rank's rows in PERMUTED order, shape [row_end - row_begin, N].
    ``row_perm``: int64 [n_rows] (VbrMatrix.row_perm).  Returns the full C [n_rows, N] in source
    row order on every rank (C[row_perm[p]] = row p of the permuted product, multiply.py:90).
    """
    world = dist.get_world_size(group)
    N = C_local.shape[1]
    max_rows = max(e - b for b, e in ranges)
    buf = torch.zeros((max_rows, N), dtype=C_local.dtype, device=C_local.device)
    buf[: C_local.shape[0]] = C_local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = torch.cat(parts, 0)
    n_rows = row_perm.numel()
    full = torch.empty((n_rows, N), dtype=C_local.dtype, device=C_local.device)
    perm = row_perm.to(C_local.device)
    for k, (b, e) in enumerate(ranges):
        if e > b:
            full[perm[b:e]] = out[k * max_rows: k * max_rows + (e - b)]
    return full


def local_rows(C_full_layout: torch.Tensor, row_perm: torch.Tensor, begin: int, end: int) -> torch.Tensor:
    """This rank's rows (permuted order) out of a full-size C that the kernel wrote in source order."""
    return C_full_layout.index_select(0, row_perm[begin:end].to(C_full_layout.device))

"""Block-row sharding of the SpMM across ranks (one process per GPU) — SURVEY.md §8(e).

Each rank owns a contiguous, work-balanced range of PERMUTED rows (whole
block-row M-tiles, ``rb_spmm_shard_range``), so it writes a disjoint set of C
rows with no data-path collective.  B is replicated.  The only collective is the
optional all-gather of C, in two forms:

* ``gather_c``: every rank's rows (in permuted order) are gathered with
  ``torch.distributed.all_gather`` (NCCL over NVLink on the GPU box, gloo in the CPU tests) and
  un-permuted in place — the baseline;
* ``FusedGather``: the SpMM epilogues store every C element of the rank's rows, already at its
  source row, into every rank's full-size C over NVLink (``rb_spmm_execute_fanout`` with the peers'
  symmetric-memory buffers), so the gather overlaps the math and there is no collective call and no
  un-permute pass; one device-side barrier orders the peers' writes before anyone reads.
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
    if buf.is_cuda and dist.get_backend(group) == "gloo":  # gloo (CPU tests / one shared GPU): stage on host
        parts = [torch.empty_like(buf, device="cpu") for _ in range(world)]
        dist.all_gather(parts, buf.cpu(), group=group)
        out = torch.cat(parts, 0).to(buf.device)
    else:
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


def shard_grouping(row_perm, row_partition, begin: int, end: int):
    """The shard [begin, end) of permuted rows as a grouping of its own: (rows, row_partition_local).

    ``rows`` are the source row ids of permuted positions begin..end-1; local row i is permuted
    position begin + i, so the shard's VBR has the identity row_perm and its C comes out in permuted
    order (what gather_c takes).  ``row_partition_local`` cuts the range at the global block-row
    boundaries (a tall block row cut by the shard keeps its rows in one local block row).  Works on
    numpy or torch inputs."""
    rp = row_partition if isinstance(row_partition, torch.Tensor) else torch.as_tensor(np.asarray(row_partition))
    rp = rp.to(torch.int64)
    inner = rp[(rp > begin) & (rp < end)] - begin
    cuts = torch.cat([torch.zeros(1, dtype=torch.int64, device=rp.device), inner,
                      torch.full((1,), end - begin, dtype=torch.int64, device=rp.device)])
    if end <= begin:
        cuts = torch.zeros(1, dtype=torch.int64, device=rp.device)
    perm = row_perm if isinstance(row_perm, torch.Tensor) else torch.as_tensor(np.asarray(row_perm))
    return perm[begin:end].to(torch.int64), cuts


def take_rows(A, rows: torch.Tensor):
    """CSR of the given source rows (in that order) of a DeviceCsr, on A's device (torch gathers)."""
    from .device import DeviceCsr

    rows = rows.to(A.row_ptr.device)
    start = A.row_ptr[rows]
    cnt = A.row_ptr[rows + 1] - start
    rp = torch.zeros(rows.numel() + 1, dtype=torch.int64, device=rows.device)
    torch.cumsum(cnt, 0, out=rp[1:])
    total = int(rp[-1].item()) if rows.numel() else 0
    idx = torch.repeat_interleave(start - rp[:-1], cnt, output_size=total) + torch.arange(total, device=rows.device)
    vals = A.values[idx] if A.values is not None else None
    return DeviceCsr(rows.numel(), A.n_cols, rp, A.col_idx[idx], vals)


def shard_vbr(dA, partition, row_perm, row_partition, precision: str, shard: int, n_shards: int, dp: int = 64):
    """This rank's own VBR: the rows of its work-balanced shard (rb_spmm_shard_range over the full
    block structure) as a sub-matrix with its own tiles, so a rank holds 1/n_shards of the tiles
    (each rank builds only its own tiles).  Returns (DeviceVbr, (begin, end), ranges)."""
    from .device import DeviceVbr

    full = DeviceVbr.build(dA, partition, row_perm, row_partition, dtypes=())  # structure only, no tiles
    rp, bp, _ = full.host_structure()
    ranges = all_ranges(rp, bp, precision, dp, n_shards)
    b, e = ranges[shard]
    rows, cuts = shard_grouping(full.row_perm64, rp, b, e)
    sub = take_rows(dA, rows)
    dv = DeviceVbr.build(sub, partition, torch.arange(e - b, dtype=torch.int64, device=rows.device), cuts,
                         dtypes=(precision,))
    dv.work_shards = n_shards  # plans size hub-row parts for a 1/n_shards share of the product
    dv.global_rows = rows.to(torch.int32).contiguous()  # output rows for the fused gather (c_rows)
    return dv, (b, e), ranges


def local_rows(C_full_layout: torch.Tensor, row_perm: torch.Tensor, begin: int, end: int) -> torch.Tensor:
    """This rank's rows (permuted order) out of a full-size C that the kernel wrote in source order."""
    return C_full_layout.index_select(0, row_perm[begin:end].to(C_full_layout.device))


def global_rows_of(row_perm, begin: int, end: int) -> torch.Tensor:
    """int32 output rows (source row ids) of permuted positions [begin, end): the c_rows a shard's
    sub-VBR passes to the fused gather (C[row_perm[p]] = row p of the permuted product, multiply.py:90)."""
    perm = row_perm if isinstance(row_perm, torch.Tensor) else torch.as_tensor(np.asarray(row_perm))
    return perm[begin:end].to(torch.int32).contiguous()


class FusedGather:
    """Full-size float32 C [n_rows, N] on every rank in symmetric memory, plus views of every peer's
    copy mapped into this process over NVLink (torch symmetric memory: P2P-mapped allocations).

    ``run(dv, B)`` multiplies this rank's sub-VBR with rb_spmm_execute_fanout: the epilogues write the
    rank's rows into its own buffer and all peers' buffers, then a device-side barrier (on the same
    stream) makes every rank's rows visible to every rank.  Afterwards ``self.C`` holds the whole
    product in source row order on every rank — what gather_c returns — with no NCCL call.
    Needs a CUDA process group whose GPUs are NVLink peers."""

    def __init__(self, n_rows: int, N: int, device, group=None):
        import torch.distributed._symmetric_memory as symm_mem

        self.group = group or dist.group.WORLD
        self.rank, self.world = dist.get_rank(self.group), dist.get_world_size(self.group)
        if self.world > 8:
            raise ValueError("fused gather supports up to 8 ranks (7 peers)")
        name = self.group.group_name
        try:  # required by older torch releases, a no-op / absent in newer ones
            symm_mem.enable_symm_mem_for_group(name)
        except Exception:  # noqa: BLE001
            pass
        self.C = symm_mem.empty((n_rows, N), dtype=torch.float32, device=device)
        self.handle = symm_mem.rendezvous(self.C, name)
        self.peers = [self.handle.get_buffer(r, (n_rows, N), torch.float32) for r in range(self.world)
                      if r != self.rank]

    def run(self, dv, B: torch.Tensor, precision: str | None = None, stream=None) -> torch.Tensor:
        rows = getattr(dv, "global_rows", None)
        dv.spmm_fanout(B, self.C, self.peers, c_rows=rows, precision=precision, stream=stream, validate=False)
        s = stream or torch.cuda.current_stream()
        with torch.cuda.stream(s):
            self.handle.barrier(channel=0)
        return self.C

"""Device-resident forms of the hot-path objects and the torch-native API.

    DeviceCsr       CSR pattern + values in HBM (int64 / float64, as CsrMatrix)
    DeviceGrouping  output of block_1sa on the device (RowGrouping arrays)
    DeviceVbr       VBR structure + padded tiles in HBM (see DESIGN.md §3 for the layout)

``block_1sa_device`` → ``DeviceVbr.build`` → ``DeviceVbr.spmm`` is the hot path
with every buffer resident in HBM; the reference-facing functions in
``blocking.py`` / ``vbr.py`` / ``multiply.py`` wrap these with host copies.
"""

from __future__ import annotations

import ctypes
import warnings
import weakref

import numpy as np
import torch

from . import _lib as L
from .types import ColumnPartition, MergePolicy, RowGroup, RowGrouping, VbrBlock


def host_tensor(a: np.ndarray) -> torch.Tensor:
    """Zero-copy CPU tensor over a (possibly read-only, frozen) numpy array; it is only ever read."""
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(np.ascontiguousarray(a))


def _i64(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.int64).contiguous()
    return host_tensor(np.asarray(x, dtype=np.int64)).to(device)


def tile_pitch(h: int) -> int:
    """Row pitch of a block row's tiles (mirrors csrc/common.cuh tile_pitch): h for h <= 8, else hp_of."""
    return h if h <= 8 else hp_of(h)


def hp_of(h: int) -> int:
    """Padded tile height (mirrors csrc/common.cuh hp_of)."""
    if h <= 16:
        return 16
    if h <= 128:
        p = 16
        while p < h:
            p <<= 1
        return p
    return (h + 127) // 128 * 128


class DeviceCsr:
    """CSR in device memory; ``row_ptr``/``col_idx`` int64, ``values`` float64."""

    def __init__(self, n_rows: int, n_cols: int, row_ptr: torch.Tensor, col_idx: torch.Tensor,
                 values: torch.Tensor | None):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_ptr, self.col_idx, self.values = row_ptr, col_idx, values

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    @classmethod
    def from_host(cls, A, device=None) -> "DeviceCsr":
        dev = device or L.require_cuda()
        vals = host_tensor(np.asarray(A.values, dtype=np.float64)).to(dev)
        return cls(A.n_rows, A.n_cols, _i64(A.row_ptr, dev), _i64(A.col_idx, dev), vals)

    # ---------------------------------------------------------------- spmm_csr comparator (rb_csr_*)
    def csr_plan(self, N: int, precision="bf16", stream=None):
        td = L.PRECISION[precision] if isinstance(precision, str) else int(precision)
        plans = self.__dict__.setdefault("_csr_plans", {})
        key = (int(N), td)
        if key not in plans:
            h = ctypes.c_void_p(0)
            L.check(L.lib().rb_csr_plan_create(self.n_rows, self.n_cols, L.ptr(self.row_ptr), int(N), td,
                                               ctypes.byref(h), L.stream_handle(stream)))
            plans[key] = h
            weakref.finalize(self, DeviceCsr._destroy_csr_plans, plans)
        return plans[key]

    @staticmethod
    def _destroy_csr_plans(plans):
        try:
            lib = L.lib()
        except Exception:  # interpreter shutdown
            return
        for h in plans.values():
            lib.rb_csr_plan_destroy(h)
        plans.clear()

    def spmm(self, B: torch.Tensor, out: torch.Tensor | None = None, precision: str | None = None,
             stream=None) -> torch.Tensor:
        """C[n_rows, N] (float32) = A @ B straight from CSR (spmm_csr, multiply.py:51-69)."""
        if B.dim() != 2 or B.shape[0] != self.n_cols:
            raise ValueError(f"dimension mismatch: {self.n_cols} vs {B.shape[0] if B.dim() == 2 else B.shape}")
        prec = precision or {torch.bfloat16: "bf16", torch.float16: "fp16", torch.float32: "fp32"}[B.dtype]
        if L.TORCH_DTYPE[L.PRECISION[prec]] != B.dtype or B.stride(1) != 1:
            raise ValueError("B must be row-major with the precision's dtype")
        N = B.shape[1]
        if out is None:
            out = torch.empty((self.n_rows, N), dtype=torch.float32, device=B.device)
        if out.dtype != torch.float32 or out.shape != (self.n_rows, N) or out.stride(1) != 1:
            raise ValueError("out must be float32 [n_rows, N], row-major")
        if N == 0 or self.n_rows == 0:
            return out
        h = self.csr_plan(N, prec, stream)
        L.check(L.lib().rb_csr_execute(h, L.ptr(self.row_ptr), L.ptr(self.col_idx), L.ptr(self.values), L.ptr(B),
                                       B.stride(0), L.ptr(out), out.stride(0), L.stream_handle(stream)))
        return out


def _boundaries(partition, n_cols: int, device) -> tuple[torch.Tensor, np.ndarray]:
    b = np.asarray(partition.boundaries if hasattr(partition, "boundaries") else partition, dtype=np.int64)
    if int(getattr(partition, "n_cols", b[-1] if b.size else 0)) != n_cols:
        raise ValueError("grouping/partition inconsistent with matrix dimensions")
    return _i64(b, device), b


class DeviceGrouping:
    """block_1sa result in device memory (int64 arrays, RowGrouping semantics)."""

    def __init__(self, n_rows, n_groups, group_of, row_perm, group_ptr, seed_size, pattern_ptr, pattern_idx):
        self.n_rows, self.n_groups = int(n_rows), int(n_groups)
        self.group_of, self.row_perm, self.group_ptr = group_of, row_perm, group_ptr
        self.seed_size, self.pattern_ptr, self.pattern_idx = seed_size, pattern_ptr, pattern_idx

    def to_host(self) -> RowGrouping:
        """Materialise the reference's RowGrouping (tuple of RowGroup, blocking.py:269-280)."""
        H = self.n_groups
        go = self.group_of.cpu().numpy()
        rp = self.row_perm.cpu().numpy()
        gp = self.group_ptr[: H + 1].cpu().numpy()
        ss = self.seed_size[:H].cpu().numpy()
        pp = self.pattern_ptr[: H + 1].cpu().numpy()
        pi = self.pattern_idx[: int(pp[-1]) if H else 0].cpu().numpy()
        groups = [RowGroup(rp[gp[g]:gp[g + 1]], pi[pp[g]:pp[g + 1]], int(ss[g])) for g in range(H)]
        return RowGrouping(go, groups, device=self)


def block_1sa_device(A: DeviceCsr, partition, policy: MergePolicy, use_compression: bool = True,
                     stream=None) -> DeviceGrouping:
    """Device block_1sa (blocking.py:283-306) through rb_block_1sa."""
    if policy.similarity not in ("jaccard", "cosine"):
        raise ValueError(f"unknown similarity {policy.similarity!r}")
    if not 0.0 <= float(policy.tau) <= 1.0:
        raise ValueError("tau must be in [0, 1]")
    dev = A.row_ptr.device
    bnd, bh = _boundaries(partition, A.n_cols, dev)
    n_seg = len(bh) - 1
    n = A.n_rows
    lib = L.lib()
    ws_bytes = ctypes.c_size_t(0)
    L.check(lib.rb_block_1sa_workspace_size(n, A.nnz, n_seg, int(bool(use_compression)), ctypes.byref(ws_bytes)))
    ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device=dev)
    group_of = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    row_perm = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    group_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    seed_size = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    pattern_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    pattern_idx = torch.empty(max(A.nnz, 1), dtype=torch.int64, device=dev)
    H = ctypes.c_int64(0)
    L.check(lib.rb_block_1sa(n, A.n_cols, A.nnz, L.ptr(A.row_ptr), L.ptr(A.col_idx), L.ptr(bnd), n_seg,
                             float(policy.tau), L.RB_COSINE if policy.similarity == "cosine" else L.RB_JACCARD,
                             int(bool(policy.bounded)), int(bool(policy.pattern_update)), int(bool(use_compression)),
                             L.ptr(ws), ws_bytes.value, L.ptr(group_of), L.ptr(row_perm), L.ptr(group_ptr),
                             L.ptr(seed_size), L.ptr(pattern_ptr), L.ptr(pattern_idx), ctypes.byref(H),
                             L.stream_handle(stream)))
    return DeviceGrouping(n, H.value, group_of[:n], row_perm[:n], group_ptr, seed_size, pattern_ptr, pattern_idx)


class DeviceVbr:
    """VBR matrix resident in HBM.

    Structure (int32): row_partition[H+1], row_perm[n], blk_ptr[H+1], blk_col[nb],
    grp_tile_row[H] (int64), col_bounds[n_seg+1].  Tiles: block t of block row g is a
    row-major tile of h_g valid rows x dp at tile row grp_tile_row[g] + t*pitch(h_g), pitch = h_g
    for h_g <= 8 else hp(h_g) (zero padding rows); one tile array per dtype.
    """

    def __init__(self):
        self._plans: dict = {}
        self.tiles: dict = {}
        self._finalizer = None

    # ---------------------------------------------------------------- build (rb_vbr_plan / emit)
    @classmethod
    def build(cls, A: DeviceCsr, partition, row_perm, row_partition, dtypes=("bf16",), stream=None) -> "DeviceVbr":
        dev = A.row_ptr.device
        self = cls()
        self.csr = A
        self.n_rows, self.n_cols = A.n_rows, A.n_cols
        self.boundaries, bh = _boundaries(partition, A.n_cols, dev)
        self.boundaries_host = bh
        self.n_seg = len(bh) - 1
        self.max_width = int(np.diff(bh).max()) if self.n_seg else 0
        self.row_perm64 = _i64(row_perm, dev)
        self.row_partition64 = _i64(row_partition, dev)
        if self.row_perm64.numel() != A.n_rows:
            raise ValueError("grouping/partition inconsistent with matrix dimensions")
        H = self.row_partition64.numel() - 1
        self.n_block_rows = H
        lib = L.lib()
        wsb = ctypes.c_size_t(0)
        L.check(lib.rb_vbr_workspace_size(A.n_rows, H, self.n_seg, ctypes.byref(wsb)))
        self._ws = torch.empty(max(1, wsb.value), dtype=torch.uint8, device=dev)
        n = A.n_rows
        self.row_perm = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.row_partition = torch.empty(H + 1, dtype=torch.int32, device=dev)
        self.blk_ptr = torch.empty(H + 1, dtype=torch.int32, device=dev)
        self.grp_tile_row = torch.empty(max(H, 1), dtype=torch.int64, device=dev)
        self.col_bounds = torch.empty(self.n_seg + 1, dtype=torch.int32, device=dev)
        nb, rows = ctypes.c_int64(0), ctypes.c_int64(0)
        L.check(lib.rb_vbr_plan(A.n_rows, A.n_cols, L.ptr(A.row_ptr), L.ptr(A.col_idx), L.ptr(self.boundaries),
                                self.n_seg, L.ptr(self.row_perm64), L.ptr(self.row_partition64), H, L.ptr(self._ws),
                                wsb.value, L.ptr(self.row_perm), L.ptr(self.row_partition), L.ptr(self.blk_ptr),
                                L.ptr(self.grp_tile_row), L.ptr(self.col_bounds), ctypes.byref(nb),
                                ctypes.byref(rows), L.stream_handle(stream)))
        self.n_blocks, self.total_tile_rows = nb.value, rows.value
        self.blk_col = torch.empty(max(self.n_blocks, 1), dtype=torch.int32, device=dev)
        self._ws_bytes = wsb.value
        self._blkcol_done = False
        for d in dtypes:
            self.tiles_for(d, stream=stream)
        if not self._blkcol_done:
            self._emit(None, L.RB_F32, self.dp_for(L.RB_F32), stream)
        return self

    def dp_for(self, tile_dtype: int) -> int:
        w = max(self.max_width, 1)
        return (w + 63) // 64 * 64 if tile_dtype in (L.RB_BF16, L.RB_F16) else (w + 3) // 4 * 4

    def _emit(self, tiles, tile_dtype, dp, stream):
        L.check(L.lib().rb_vbr_emit(self.n_rows, L.ptr(self.csr.row_ptr), L.ptr(self.csr.col_idx),
                                    L.ptr(self.csr.values), L.ptr(self.boundaries), self.n_seg, self.n_block_rows,
                                    L.ptr(self._ws), self._ws_bytes, L.ptr(self.row_perm), L.ptr(self.row_partition),
                                    L.ptr(self.blk_ptr), L.ptr(self.grp_tile_row), L.ptr(self.blk_col),
                                    L.ptr(tiles), tile_dtype, dp, self.total_tile_rows if tiles is not None else 0,
                                    L.stream_handle(stream)))
        self._blkcol_done = True

    def tiles_for(self, precision, stream=None) -> tuple[torch.Tensor, int]:
        """(tiles, dp) of the given precision ("bf16"/"fp16"/"fp32" or an RB_* code), built on demand."""
        td = L.PRECISION[precision] if isinstance(precision, str) else int(precision)
        if td not in self.tiles:
            dp = self.dp_for(td)
            t = torch.empty((max(self.total_tile_rows, 1), dp), dtype=L.TORCH_DTYPE[td], device=self.blk_ptr.device)
            self._emit(t, td, dp, stream)
            self.tiles[td] = (t, dp)
        return self.tiles[td]

    # ---------------------------------------------------------------- SpMM (rb_spmm_*)
    def compact(self, td: int, h_max: int, stream=None):
        """Compact payloads of the block rows with h <= h_max (rb_vbr_compact_*), per tile dtype:
        (cmp_ptr int64[n_rows+1], cmp_col int32, cmp_val float32) or None if no row qualifies."""
        cache = self.__dict__.setdefault("_compact", {})
        key = (td, h_max)
        if key not in cache:
            lib = L.lib()
            dev = self.blk_ptr.device
            ptr = torch.empty(self.n_rows + 1, dtype=torch.int64, device=dev)
            total = ctypes.c_int64(0)
            L.check(lib.rb_vbr_compact_count(self.n_rows, L.ptr(self.csr.row_ptr), L.ptr(self.row_perm),
                                             L.ptr(self.row_partition), self.n_block_rows, int(h_max), L.ptr(ptr),
                                             ctypes.byref(total), L.stream_handle(stream)))
            if total.value == 0:
                cache[key] = None
            else:
                col = torch.empty(total.value, dtype=torch.int32, device=dev)
                val = torch.empty(total.value, dtype=torch.float32, device=dev)
                L.check(lib.rb_vbr_compact_emit(self.n_rows, L.ptr(self.csr.row_ptr), L.ptr(self.csr.col_idx),
                                                L.ptr(self.csr.values), L.ptr(self.row_perm), L.ptr(ptr), td,
                                                L.ptr(col), L.ptr(val), L.stream_handle(stream)))
                cache[key] = (ptr, col, val)
        return cache[key]

    def _struct(self, td: int) -> L.VbrDevice:
        from . import config

        t, dp = self.tiles_for(td)
        s = L.VbrDevice(self.n_rows, self.n_cols, self.n_block_rows, self.n_blocks, self.n_seg,
                        self.total_tile_rows, dp, td, self.row_partition.data_ptr(), self.row_perm.data_ptr(),
                        self.blk_ptr.data_ptr(), self.blk_col.data_ptr(), self.grp_tile_row.data_ptr(),
                        self.col_bounds.data_ptr(), t.data_ptr())
        h_max = config.compact_h()
        if h_max > 0 and td in (L.RB_BF16, L.RB_F16, L.RB_F32) and self.csr.values is not None:
            c = self.compact(td, h_max)
            if c is not None:
                s.cmp_ptr, s.cmp_col, s.cmp_val, s.cmp_h = c[0].data_ptr(), c[1].data_ptr(), c[2].data_ptr(), h_max
        return s

    # ---------------------------------------------------------------- 2:4 sparse form (rb_sparse24_*)
    def sparse24(self, precision="bf16", stream=None) -> "L.Sparse24Device":
        """Compressed 2:4 form of the tall block rows (+ residual CSR), built once per dtype."""
        td = L.PRECISION[precision] if isinstance(precision, str) else int(precision)
        cache = self.__dict__.setdefault("_sp24", {})
        if td in cache:
            return cache[td][0]
        lib = L.lib()
        dev = self.blk_ptr.device
        s = self._struct(td)
        H = self.n_block_rows
        spr_host = np.zeros(max(H, 1), np.int64)
        total, n_tall = ctypes.c_int64(0), ctypes.c_int64(0)
        L.check(lib.rb_sparse24_layout(ctypes.byref(s), ctypes.c_void_p(spr_host.ctypes.data), ctypes.byref(total),
                                       ctypes.byref(n_tall), L.stream_handle(stream)))
        rp = self.row_partition.cpu().numpy().astype(np.int64)
        tall_g = np.flatnonzero(spr_host[:H] >= 0).astype(np.int32)
        hs = ((np.diff(rp)[tall_g] + 255) // 256 * 256).astype(np.int64)
        tbase = np.concatenate([[0], np.cumsum(hs)]).astype(np.int64)
        keep = {
            "sp_tile_row": torch.from_numpy(spr_host).to(dev),
            "tall_g": torch.from_numpy(tall_g if len(tall_g) else np.zeros(1, np.int32)).to(dev),
            "tbase": torch.from_numpy(tbase).to(dev),
            "tiles": torch.zeros((max(total.value, 1), 64), dtype=L.TORCH_DTYPE[td], device=dev),
            "meta": torch.zeros(max(total.value, 1) * 8, dtype=torch.int32, device=dev),
            "res_ptr": torch.zeros(self.n_rows + 1, dtype=torch.int64, device=dev),
        }
        wsb = ctypes.c_size_t(0)
        L.check(lib.rb_sparse24_workspace_size(self.n_rows, total.value, ctypes.byref(wsb)))
        ws = torch.empty(max(1, wsb.value), dtype=torch.uint8, device=dev)
        n_res = ctypes.c_int64(0)
        args = lambda tiles, meta, rc, rv, cap: (  # noqa: E731
            ctypes.byref(s), L.ptr(keep["sp_tile_row"]), L.ptr(keep["tall_g"]), L.ptr(keep["tbase"]), len(tall_g),
            int(tbase[-1]), total.value, L.ptr(ws), wsb.value, tiles, meta, L.ptr(keep["res_ptr"]), rc, rv, cap,
            ctypes.byref(n_res), L.stream_handle(stream))
        L.check(lib.rb_sparse24_emit(*args(None, None, None, None, 0)))  # residual counts
        keep["res_col"] = torch.empty(max(n_res.value, 1), dtype=torch.int32, device=dev)
        keep["res_val"] = torch.empty(max(n_res.value, 1), dtype=torch.float32, device=dev)
        L.check(lib.rb_sparse24_emit(*args(L.ptr(keep["tiles"]), L.ptr(keep["meta"]), L.ptr(keep["res_col"]),
                                           L.ptr(keep["res_val"]), n_res.value)))
        sp = L.Sparse24Device(keep["tiles"].data_ptr(), keep["meta"].data_ptr(), keep["sp_tile_row"].data_ptr(),
                              total.value, keep["res_ptr"].data_ptr(), keep["res_col"].data_ptr(),
                              keep["res_val"].data_ptr(), n_res.value)
        cache[td] = (sp, keep)
        return sp

    def plan(self, N: int, precision="bf16", shard: int = 0, n_shards: int = 1, stream=None,
             sparse24: bool | None = None):
        from . import config

        td = L.PRECISION[precision] if isinstance(precision, str) else int(precision)
        sp24 = (config.default_sparse24() if sparse24 is None else bool(sparse24)) and td in (L.RB_BF16, L.RB_F16)
        key = (int(N), td, int(shard), int(n_shards), sp24, config.compact_h())
        if key not in self._plans:
            s = self._struct(td)
            h = ctypes.c_void_p(0)
            work = max(int(n_shards), int(getattr(self, "work_shards", 1)))  # set by dist.shard_vbr
            L.check(L.lib().rb_spmm_plan_create_ex(ctypes.byref(s), int(N), td, int(shard), int(n_shards), work,
                                                   ctypes.byref(h), L.stream_handle(stream)))
            if sp24:
                try:
                    L.check(L.lib().rb_spmm_plan_attach_sparse24(h, ctypes.byref(self.sparse24(td, stream)),
                                                                 L.stream_handle(stream)))
                except Exception:
                    L.lib().rb_spmm_plan_destroy(h)
                    raise
            self._plans[key] = h
            if self._finalizer is None:
                self._finalizer = weakref.finalize(self, DeviceVbr._destroy_plans, self._plans)
        return self._plans[key]

    @staticmethod
    def _destroy_plans(plans):
        try:
            lib = L.lib()
        except Exception:  # interpreter shutdown
            return
        for h in plans.values():
            lib.rb_spmm_plan_destroy(h)
        plans.clear()

    def plan_info(self, N: int, precision="bf16", shard: int = 0, n_shards: int = 1, sparse24=None) -> dict:
        info = L.SpmmInfo()
        L.check(L.lib().rb_spmm_plan_info(self.plan(N, precision, shard, n_shards, sparse24=sparse24),
                                          ctypes.byref(info)))
        return {f: getattr(info, f) for f, _ in L.SpmmInfo._fields_}

    def spmm(self, B: torch.Tensor, out: torch.Tensor | None = None, precision: str | None = None,
             shard: int = 0, n_shards: int = 1, stream=None, sparse24: bool | None = None) -> torch.Tensor:
        """C[n_rows, N] = A @ B on the device: float32 for B bf16/fp16/fp32 (row stride a multiple of 8
        elements for 16-bit types), float64 for B float64 (the fp64 path).  ``out`` rows not owned by
        ``shard`` are untouched."""
        if B.dim() != 2 or B.shape[0] != self.n_cols:
            raise ValueError(f"dimension mismatch: {self.n_cols} vs {B.shape[0] if B.dim() == 2 else B.shape}")
        prec = precision or {torch.bfloat16: "bf16", torch.float16: "fp16", torch.float32: "fp32",
                             torch.float64: "fp64"}[B.dtype]
        if L.TORCH_DTYPE[L.PRECISION[prec]] != B.dtype:
            raise ValueError(f"B dtype {B.dtype} does not match precision {prec}")
        N = B.shape[1]
        if B.stride(1) != 1:
            raise ValueError("B must be row-major (stride(1) == 1)")
        cdt = torch.float64 if prec == "fp64" else torch.float32
        if out is None:
            out = torch.empty((self.n_rows, N), dtype=cdt, device=B.device)
        if out.dtype != cdt or out.shape != (self.n_rows, N) or out.stride(1) != 1:
            raise ValueError(f"out must be {cdt} [n_rows, N], row-major")
        if N == 0 or self.n_rows == 0:
            return out
        h = self.plan(N, prec, shard, n_shards, stream, sparse24=sparse24)
        run = L.lib().rb_spmm_execute_f64 if prec == "fp64" else L.lib().rb_spmm_execute
        L.check(run(h, L.ptr(B), B.stride(0), L.ptr(out), out.stride(0), L.stream_handle(stream)))
        return out

    def spmm_fanout(self, B: torch.Tensor, out: torch.Tensor, peers=(), c_rows: torch.Tensor | None = None,
                    precision: str | None = None, shard: int = 0, n_shards: int = 1, stream=None,
                    validate: bool = True) -> torch.Tensor:
        """Fused all-gather (rb_spmm_execute_fanout): C = A @ B into ``out`` (float32) and, by the
        same epilogue stores, into every tensor of ``peers`` (the other ranks' full-size C mapped over
        NVLink — dist.FusedGather — or any device buffers shaped like ``out``).  ``c_rows``: int32
        device [n_rows], the output row of each permuted row (None: row_perm, out is [n_rows, N]);
        a rank's sub-VBR passes its shard's global source rows (dist.shard_vbr sets
        ``global_rows``), so ``out`` / ``peers`` are the full [n_rows_global, N] C."""
        if B.dim() != 2 or B.shape[0] != self.n_cols:
            raise ValueError(f"dimension mismatch: {self.n_cols} vs {B.shape[0] if B.dim() == 2 else B.shape}")
        prec = precision or {torch.bfloat16: "bf16", torch.float16: "fp16", torch.float32: "fp32"}[B.dtype]
        if prec == "fp64":
            raise ValueError("fan-out writes float32 C (no fp64 path)")
        if L.TORCH_DTYPE[L.PRECISION[prec]] != B.dtype or B.stride(1) != 1:
            raise ValueError("B must be row-major with the precision's dtype")
        N = B.shape[1]
        peers = list(peers)
        if len(peers) > 7:
            raise ValueError("at most 7 peers (8 ranks)")
        for t in [out] + peers:
            if (t.dtype != torch.float32 or t.dim() != 2 or t.shape != out.shape or t.stride() != out.stride()
                    or t.stride(1) != 1 or out.shape[1] != N):
                raise ValueError("out / peers must be float32 [rows, N] row-major buffers of one layout")
        if c_rows is None:
            if out.shape[0] != self.n_rows:
                raise ValueError("out must have n_rows rows when c_rows is None")
        else:
            if c_rows.dtype != torch.int32 or c_rows.numel() != self.n_rows or not c_rows.is_contiguous():
                raise ValueError("c_rows must be a contiguous int32 tensor of n_rows entries")
            if validate and self.n_rows and not (0 <= int(c_rows.min()) and int(c_rows.max()) < out.shape[0]):
                raise ValueError("c_rows out of range of out")
        if N == 0 or self.n_rows == 0:
            return out
        h = self.plan(N, prec, shard, n_shards, stream)
        arr = (ctypes.c_void_p * max(1, len(peers)))(*[L.ptr(t) for t in peers])
        L.check(L.lib().rb_spmm_execute_fanout(h, L.ptr(B), B.stride(0), L.ptr(out), out.stride(0), arr, len(peers),
                                               L.ptr(c_rows) if c_rows is not None else None,
                                               L.stream_handle(stream)))
        return out

    # ---------------------------------------------------------------- reference-format views
    def host_structure(self):
        rp = self.row_partition.cpu().numpy().astype(np.int64)
        bp = self.blk_ptr.cpu().numpy().astype(np.int64)
        bc = self.blk_col[: self.n_blocks].cpu().numpy().astype(np.int64)
        return rp, bp, bc

    def stored_area(self) -> int:
        rp, bp, bc = self.host_structure()
        widths = np.diff(self.boundaries_host)
        heights = np.diff(rp)
        blk_h = np.repeat(heights, np.diff(bp))
        return int(np.sum(blk_h * widths[bc])) if len(bc) else 0

    def host_block_rows(self) -> tuple:
        """float64 payloads (vbr.py:113-123) via a float64 tile emission on the device."""
        t, dp = self.tiles_for(L.RB_F64)
        tiles = t.cpu().numpy()
        del self.tiles[L.RB_F64]
        rp, bp, bc = self.host_structure()
        tr = self.grp_tile_row[: self.n_block_rows].cpu().numpy()
        widths = np.diff(self.boundaries_host)
        out = []
        for g in range(self.n_block_rows):
            h = int(rp[g + 1] - rp[g])
            hp = tile_pitch(h)
            base = int(tr[g])
            out.append(tuple(VbrBlock(int(bc[k]), tiles[base + (k - bp[g]) * hp: base + (k - bp[g]) * hp + h,
                                                          : int(widths[bc[k]])])
                             for k in range(int(bp[g]), int(bp[g + 1]))))
        return tuple(out)

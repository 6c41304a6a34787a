"""Blocking quality on the device — drop-in for rowblock.metrics (metrics.py:1-216).

Same dataclasses, functions, defaults and errors as the reference:

    blocking_stats(A, grouping, partition, tau=None, check_bound=False) -> BlockingStats   (59-95)
    blocking_curve(A, partition, taus, policy, use_compression, jobs, meta) -> BlockingCurve (106-130)
    curve_select(curve, at_height=None, at_density=None) -> (tau, BlockingStats)          (133-147)
    verify_density_bound(A, grouping, partition, tau) -> DensityReport                    (178-216)

The per-group reductions (stored columns, element nnz, distinct-segment counts) and the exact
rational density tests run in one CUDA kernel (csrc/stats.cu, rb_group_stats) on the grouping's
device arrays; blocking_curve runs 1-SA on the device once per tau.  The 1-SA kernel is a persistent
grid that owns its GPU, so with ``jobs != 1`` the points run concurrently across the visible GPUs
(one host thread per device), and sequentially on any one device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from fractions import Fraction

import numpy as np
import torch

from . import _lib as L
from .device import DeviceCsr, DeviceGrouping, _boundaries, _i64, block_1sa_device
from .types import ColumnPartition, MergePolicy

__all__ = ["BlockingStats", "BlockingCurve", "GroupDensity", "DensityReport", "blocking_stats", "blocking_curve",
           "curve_select", "verify_density_bound", "group_stats_device"]


@dataclass(frozen=True)
class BlockingStats:
    """Quality numbers for one blocking of one matrix (metrics.py:31-45)."""

    rho_prime: float
    delta_h_prime: float
    n_groups: int
    n_stored_blocks: int
    fill_in: int
    nnz: int
    stored_area: int
    group_mean_height: float
    tau: float | None = None
    density_bound_ok: bool | None = None


@dataclass(frozen=True)
class BlockingCurve:
    """Stats per tau, ascending (metrics.py:48-56)."""

    points: tuple
    meta: dict

    def taus(self):
        return [t for t, _ in self.points]


@dataclass(frozen=True)
class GroupDensity:
    """Per-group verdict of the density verifier (metrics.py:150-162)."""

    group: int
    n_rows: int
    pattern_size: int
    stored_cols: int
    element_nnz: int
    quotient_nnz: int
    element_density: float
    quotient_density: float
    element_ok: bool
    quotient_ok: bool


@dataclass(frozen=True)
class DensityReport:
    groups: tuple
    element_bound: float
    quotient_bound: float
    all_ok: bool

    @property
    def n_violations(self) -> int:
        return sum(1 for g in self.groups if not (g.element_ok and g.quotient_ok))


# ------------------------------------------------------------------------------------------ device


def _device_inputs(A, grouping):
    """(DeviceCsr, DeviceGrouping-like arrays) for a host or device grouping."""
    dg = getattr(grouping, "device", None) if not isinstance(grouping, DeviceGrouping) else grouping
    if isinstance(A, DeviceCsr):
        dA = A
    elif dg is not None and getattr(dg, "source", None) is A and getattr(dg, "csr", None) is not None:
        dA = dg.csr
    else:
        dA = DeviceCsr.from_host(A)
    dev = dA.row_ptr.device
    if dg is not None and dg.n_rows == dA.n_rows:
        H = dg.n_groups
        return dA, H, dg.row_perm, dg.group_ptr[: H + 1], dg.pattern_ptr[: H + 1], dg.pattern_idx
    groups = grouping.groups
    H = len(groups)
    rows = np.concatenate([np.asarray(g.rows, np.int64) for g in groups]) if H else np.zeros(0, np.int64)
    gp = np.zeros(H + 1, np.int64)
    np.cumsum([len(g.rows) for g in groups], out=gp[1:])
    pats = np.concatenate([np.asarray(g.pattern, np.int64) for g in groups]) if H else np.zeros(0, np.int64)
    pp = np.zeros(H + 1, np.int64)
    np.cumsum([len(g.pattern) for g in groups], out=pp[1:])
    return dA, H, _i64(rows, dev), _i64(gp, dev), _i64(pp, dev), _i64(pats if len(pats) else np.zeros(1, np.int64), dev)


def group_stats_device(A, grouping, partition, tau: float = 0.0, stream=None) -> dict:
    """Per-group device arrays + totals from rb_group_stats (one kernel, grouping stays in HBM)."""
    dA, H, row_perm, group_ptr, pattern_ptr, pattern_idx = _device_inputs(A, grouping)
    dev = dA.row_ptr.device
    bnd, bh = _boundaries(partition, dA.n_cols, dev)
    n_seg = len(bh) - 1
    lib = L.lib()
    wsb = ctypes.c_size_t(0)
    L.check(lib.rb_group_stats_workspace_size(n_seg, ctypes.byref(wsb)))
    ws = torch.empty(max(1, wsb.value), dtype=torch.uint8, device=dev)
    out = {k: torch.empty(max(H, 1), dtype=torch.int64, device=dev)
           for k in ("stored_cols", "element_nnz", "quotient_nnz")}
    ok = torch.empty(max(H, 1), dtype=torch.uint8, device=dev)
    tot = [ctypes.c_int64(0) for _ in range(4)]
    L.check(lib.rb_group_stats(dA.n_rows, dA.n_cols, L.ptr(dA.row_ptr), L.ptr(dA.col_idx), L.ptr(bnd), n_seg,
                               L.ptr(row_perm), L.ptr(group_ptr), L.ptr(pattern_ptr), L.ptr(pattern_idx), H,
                               float(tau), L.ptr(ws), wsb.value, L.ptr(out["stored_cols"]),
                               L.ptr(out["element_nnz"]), L.ptr(out["quotient_nnz"]), L.ptr(ok),
                               *[ctypes.byref(t) for t in tot], L.stream_handle(stream)))
    res = {k: v[:H] for k, v in out.items()}
    res.update(ok=ok[:H], heights=(group_ptr[1:] - group_ptr[:-1])[:H],
               pattern_sizes=(pattern_ptr[1:] - pattern_ptr[:-1])[:H], n_groups=H, nnz=dA.nnz,
               stored_area=tot[0].value, n_blocks=tot[1].value, height_sum=tot[2].value,
               n_violations=tot[3].value)
    return res


# ------------------------------------------------------------------------------------------ API


def blocking_stats(A, grouping, partition: ColumnPartition, tau: float | None = None,
                   check_bound: bool = False) -> BlockingStats:
    """Density / height / fill-in of a blocking (metrics.py:59-95), reduced on the device."""
    nnz = A.nnz
    if nnz == 0:
        raise ValueError("blocking stats are undefined for an empty matrix")
    if check_bound and tau is None:
        raise ValueError("check_bound requires tau")
    s = group_stats_device(A, grouping, partition, tau if (check_bound and tau is not None) else 0.0)
    H = s["n_groups"]
    area, n_blocks = s["stored_area"], s["n_blocks"]
    return BlockingStats(
        rho_prime=nnz / area,
        delta_h_prime=s["height_sum"] / n_blocks if n_blocks else 0.0,
        n_groups=H,
        n_stored_blocks=n_blocks,
        fill_in=area - nnz,
        nnz=nnz,
        stored_area=area,
        group_mean_height=float(s["heights"].cpu().numpy().mean()) if H else 0.0,
        tau=tau,
        density_bound_ok=(s["n_violations"] == 0) if check_bound else None,
    )


def blocking_curve(A, partition: ColumnPartition, taus, policy: MergePolicy = MergePolicy(),
                   use_compression: bool = True, jobs: int = 1, meta: dict | None = None,
                   devices=None) -> BlockingCurve:
    """1-SA + stats once per tau on the same input (metrics.py:106-130); points ordered by tau.

    The reference spreads the points over ``jobs`` worker processes (metrics.py:122).  Here every
    point is one device 1-SA (a grid-wide persistent kernel that occupies a whole GPU), so points run
    concurrently across GPUs: with ``jobs != 1`` they are dealt round robin to ``devices`` (default:
    every visible GPU), one host thread per device, each device holding its own copy of A.  Points
    that share a device run one after another on it.  Results are identical to the sequential run
    (the 1-SA is deterministic)."""
    import threading
    from concurrent.futures import ThreadPoolExecutor

    import torch

    taus = [float(t) for t in taus]
    if not taus or any(not 0.0 <= t <= 1.0 for t in taus):
        raise ValueError("taus must be non-empty and within [0, 1]")
    if any(b <= a for a, b in zip(taus, taus[1:])):
        raise ValueError("taus must be strictly increasing")
    if devices is None:
        devices = list(range(torch.cuda.device_count())) if jobs != 1 else [None]
    devices = list(devices) or [None]
    src = A if isinstance(A, DeviceCsr) else None
    copies, locks = {}, {d: threading.Lock() for d in devices}

    def csr_on(d):
        if d not in copies:
            if src is not None and (d is None or src.row_ptr.device == torch.device("cuda", d)):
                copies[d] = src
            elif src is not None:
                dev = torch.device("cuda", d)
                copies[d] = DeviceCsr(src.n_rows, src.n_cols, src.row_ptr.to(dev), src.col_idx.to(dev),
                                      None if src.values is None else src.values.to(dev))
            else:
                copies[d] = DeviceCsr.from_host(A, None if d is None else torch.device("cuda", d))
        return copies[d]

    def point(k):
        d = devices[k % len(devices)]
        with locks[d]:
            if d is not None:
                torch.cuda.set_device(d)
            dA_d = csr_on(d)
            t = taus[k]
            p = MergePolicy(similarity=policy.similarity, tau=t, bounded=policy.bounded,
                            pattern_update=policy.pattern_update)
            dg = block_1sa_device(dA_d, partition, p, use_compression)
            return t, blocking_stats(dA_d, dg, partition, tau=t, check_bound=policy.bounded)

    if len(devices) == 1:
        points = [point(k) for k in range(len(taus))]
    else:
        with ThreadPoolExecutor(max_workers=len(devices)) as ex:
            points = list(ex.map(point, range(len(taus))))
    dA = csr_on(devices[0])
    base = {"n_rows": dA.n_rows, "n_cols": dA.n_cols, "nnz": dA.nnz}
    if meta:
        base.update(meta)
    return BlockingCurve(tuple(points), base)


def curve_select(curve: BlockingCurve, at_height: float | None = None, at_density: float | None = None):
    """Curve point closest to the target height (or density); ties go to the larger tau
    (metrics.py:133-147)."""
    if (at_height is None) == (at_density is None):
        raise ValueError("pass exactly one of at_height / at_density")
    if not curve.points:
        raise ValueError("empty curve")
    best = None
    best_key = None
    for tau, stats in curve.points:
        key = (abs(stats.delta_h_prime - at_height) if at_height is not None
               else abs(stats.rho_prime - at_density))
        if best_key is None or key <= best_key:
            best, best_key = (tau, stats), key
    return best


def verify_density_bound(A, grouping, partition: ColumnPartition, tau: float) -> DensityReport:
    """Guaranteed density of every group of a bounded-policy blocking (metrics.py:178-216); the
    exact rational tests run on the device."""
    max_w = partition.max_width if partition.n_segments else 1
    f_tau = Fraction(float(tau))
    elem_bound = f_tau / (2 * max_w)
    quot_bound = f_tau / 2
    s = group_stats_device(A, grouping, partition, float(tau))
    H = s["n_groups"]
    h = s["heights"].cpu().numpy()
    lam = s["pattern_sizes"].cpu().numpy()
    sc = s["stored_cols"].cpu().numpy()
    ke = s["element_nnz"].cpu().numpy()
    kq = s["quotient_nnz"].cpu().numpy()
    ok = s["ok"].cpu().numpy()
    checks = []
    for g in range(H):
        if lam[g] == 0:
            checks.append(GroupDensity(g, int(h[g]), 0, 0, 0, 0, 1.0, 1.0, True, True))
            continue
        checks.append(GroupDensity(g, int(h[g]), int(lam[g]), int(sc[g]), int(ke[g]), int(kq[g]),
                                   int(ke[g]) / (int(h[g]) * int(sc[g])), int(kq[g]) / (int(h[g]) * int(lam[g])),
                                   bool(ok[g] & 1), bool(ok[g] & 2)))
    return DensityReport(tuple(checks), float(elem_bound), float(quot_bound), s["n_violations"] == 0)

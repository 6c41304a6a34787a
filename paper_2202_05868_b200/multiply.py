"""spmm_vbr — drop-in for rowblock.multiply.spmm_vbr (multiply.py:72-97) on the GPU.

C = A·B on B200 tensor cores (tcgen05, bf16/fp16 inputs, fp32 accumulate) or
the fp32 check path, with C rows written back in the source row order
(multiply.py:90).  Returns the reference's float64 DenseMatrix.  ``threads`` is
accepted for signature compatibility and ignored (the GPU kernel's result does
not depend on it, as the reference's does not, multiply.py:1-5).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from . import config
from .device import host_tensor
from .types import DenseMatrix
from .vbr import device_vbr_of

__all__ = ["spmm_vbr", "spmm_vbr_many", "spmm_vbr_device", "spmm_csr", "upload_dense", "SpmmPipeline",
           "pinned_dense"]


NONFINITE_B = ("B contains NaN or Inf: the reference propagates them through the dense block payloads "
               "(multiply.py:89, zeros included), which the tensor-core / fp32 paths do not reproduce, so "
               "they refuse; precision='fp64' reproduces the reference's propagation")


def upload_dense(B, precision: str, device=None, nonfinite: torch.Tensor | None = None) -> torch.Tensor:
    """Host float64 [K, N] → device tensor of the kernel dtype with a 16-byte aligned row stride.
    ``nonfinite``: optional device int32[1] (zeroed by the caller) set to 1 if B holds NaN / Inf."""
    dev = device or L.require_cuda()
    a = np.ascontiguousarray(np.asarray(B.data if hasattr(B, "data") else B, dtype=np.float64))
    K, N = a.shape
    td = L.PRECISION[precision]
    ld = (N + 7) // 8 * 8
    src = host_tensor(a).to(dev)
    buf = torch.empty((K, ld), dtype=L.TORCH_DTYPE[td], device=dev)
    flag = L.ptr(nonfinite) if nonfinite is not None else None
    L.check(L.lib().rb_convert_f64_checked(L.ptr(src), K, N, N, L.ptr(buf), td, ld, flag, L.stream_handle()))
    return buf[:, :N]


def spmm_vbr_device(V, B: torch.Tensor, out=None, precision=None) -> torch.Tensor:
    """Torch-native entry: V (our VbrMatrix or DeviceVbr), B device tensor → fp32 device C."""
    dv = V if hasattr(V, "spmm") else device_vbr_of(V)
    return dv.spmm(B, out=out, precision=precision)


def spmm_csr(A, B, threads: int = 1, *, precision: str | None = None) -> DenseMatrix:
    """Sparse-baseline product straight from CSR (multiply.py:51-69) on the GPU (csrc/csr.cu), the
    comparator the paper measures VBR against; float64 DenseMatrix result, empty rows exact 0."""
    from .device import DeviceCsr

    if A.n_cols != B.n_rows:
        raise ValueError(f"dimension mismatch: {A.n_cols} vs {B.n_rows}")
    prec = precision or config.default_precision()
    N = B.n_cols
    if A.n_rows == 0 or N == 0:
        return DenseMatrix(A.n_rows, N, np.zeros((A.n_rows, N)))
    dA = A if isinstance(A, DeviceCsr) else DeviceCsr.from_host(A)
    C32 = dA.spmm(upload_dense(B, prec), precision=prec)
    C64 = torch.empty((A.n_rows, N), dtype=torch.float64, device=C32.device)
    L.check(L.lib().rb_widen_f32(L.ptr(C32), A.n_rows, N, N, L.ptr(C64), N, L.stream_handle()))
    return DenseMatrix(A.n_rows, N, C64.cpu().numpy())


def spmm_vbr(V, B, threads: int = 1, *, precision: str | None = None) -> DenseMatrix:
    """Block-based product with un-permute (multiply.py:72-97); float64 DenseMatrix result."""
    if V.n_cols != B.n_rows:
        raise ValueError(f"dimension mismatch: {V.n_cols} vs {B.n_rows}")
    from . import _forkproxy
    if _forkproxy.in_bad_fork():  # forked pool worker of a CUDA parent: run in a spawned helper
        return _forkproxy.call("spmm_vbr", V, B, threads, precision=precision)
    prec = precision or config.default_precision()
    dv = device_vbr_of(V)
    N = B.n_cols
    if V.n_rows == 0 or N == 0:
        return DenseMatrix(V.n_rows, N, np.zeros((V.n_rows, N)))
    bad = torch.zeros(1, dtype=torch.int32, device=L.require_cuda())
    Bd = upload_dense(B, prec, nonfinite=bad)
    if prec == "fp64":  # float64 end to end; non-finite B propagates as in the reference
        return DenseMatrix(V.n_rows, N, dv.spmm(Bd, precision=prec).cpu().numpy())
    C32 = dv.spmm(Bd, precision=prec)
    C64 = torch.empty((V.n_rows, N), dtype=torch.float64, device=C32.device)
    L.check(L.lib().rb_widen_f32(L.ptr(C32), V.n_rows, N, N, L.ptr(C64), N, L.stream_handle()))
    C = C64.cpu().numpy()  # synchronises: the flag below is final
    if int(bad.item()):
        raise ValueError(NONFINITE_B)
    return DenseMatrix(V.n_rows, N, C)


def pinned_dense(n_rows: int, n_cols: int) -> torch.Tensor:
    """A page-locked float64 host buffer (the fast H2D/D2H source / destination for SpmmPipeline)."""
    return torch.empty((n_rows, n_cols), dtype=torch.float64).pin_memory()


class SpmmPipeline:
    """Streams many products C_k = A·B_k through one VBR plan with host float64 B_k / C_k.

    Three CUDA streams and ``depth`` device buffer sets overlap step k+1's host→device copy of B
    (+ conversion to the kernel dtype), step k's SpMM (+ widening to float64) and step k-1's
    device→host copy of C: the PCIe copy engines run both directions at once and the tensor-core
    kernel hides behind them.  Every step still moves its whole B in and its whole C out; results
    are bit-identical to ``spmm_vbr`` (same plan, same kernels).  A pipeline must not be driven
    from two host threads at once."""

    def __init__(self, V, N: int, precision: str | None = None, depth: int = 2, device=None):
        self.dv = V if hasattr(V, "spmm") else device_vbr_of(V)
        self.prec = precision or config.default_precision()
        self.td = L.PRECISION[self.prec]
        dev = device or L.require_cuda()
        self.K, self.M, self.N = self.dv.n_cols, self.dv.n_rows, int(N)
        self.ld = (self.N + 7) // 8 * 8
        self.depth = depth
        self.b64 = [torch.empty((self.K, self.N), dtype=torch.float64, device=dev) for _ in range(depth)]
        self.bk = [torch.empty((self.K, self.ld), dtype=L.TORCH_DTYPE[self.td], device=dev) for _ in range(depth)]
        self.c64 = [torch.empty((self.M, self.N), dtype=torch.float64, device=dev) for _ in range(depth)]
        self.c32 = (self.c64 if self.prec == "fp64" else
                    [torch.empty((self.M, self.N), dtype=torch.float32, device=dev) for _ in range(depth)])
        self.s_in, self.s_comp, self.s_out = (torch.cuda.Stream(dev) for _ in range(3))
        mk = lambda: [torch.cuda.Event() for _ in range(depth)]  # noqa: E731
        self.ev_in, self.ev_comp, self.ev_out = mk(), mk(), mk()
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=dev)  # set by any step's B conversion
        self.used = [False] * depth
        self.dv.plan(self.N, self.prec, stream=self.s_comp)  # plan creation outside the steady state

    def step(self, k: int, B_host: torch.Tensor, C_host: torch.Tensor) -> None:
        """Enqueue product k: B_host [K, N] float64 (pinned for full speed) → C_host [M, N] float64."""
        if B_host.shape != (self.K, self.N) or C_host.shape != (self.M, self.N):
            raise ValueError("dimension mismatch")
        i = k % self.depth
        lib = L.lib()
        with torch.cuda.stream(self.s_in):
            if self.used[i]:
                self.s_in.wait_event(self.ev_comp[i])  # buffers of step k - depth consumed
            self.b64[i].copy_(B_host, non_blocking=True)
            L.check(lib.rb_convert_f64_checked(L.ptr(self.b64[i]), self.K, self.N, self.N, L.ptr(self.bk[i]),
                                               self.td, self.ld, L.ptr(self.nonfinite), L.stream_handle(self.s_in)))
            self.ev_in[i].record(self.s_in)
        with torch.cuda.stream(self.s_comp):
            self.s_comp.wait_event(self.ev_in[i])
            if self.used[i]:
                self.s_comp.wait_event(self.ev_out[i])  # C buffers of step k - depth copied out
            self.dv.spmm(self.bk[i][:, :self.N], out=self.c32[i], precision=self.prec, stream=self.s_comp)
            if self.prec != "fp64":
                L.check(lib.rb_widen_f32(L.ptr(self.c32[i]), self.M, self.N, self.N, L.ptr(self.c64[i]), self.N,
                                         L.stream_handle(self.s_comp)))
            self.ev_comp[i].record(self.s_comp)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.ev_comp[i])
            C_host.copy_(self.c64[i], non_blocking=True)
            self.ev_out[i].record(self.s_out)
        self.used[i] = True

    def synchronize(self) -> None:
        self.s_out.synchronize()

    def check_finite(self) -> None:
        """Raise ValueError if any B converted so far held NaN / Inf (see NONFINITE_B); the fp64
        path propagates them instead, as the reference does."""
        self.s_in.synchronize()
        if self.prec != "fp64" and int(self.nonfinite.item()):
            raise ValueError(NONFINITE_B)


def spmm_vbr_many(V, Bs, threads: int = 1, *, precision: str | None = None, out=None) -> list:
    """spmm_vbr over a sequence of right-hand sides, pipelined (SpmmPipeline); returns float64
    DenseMatrix results in order.  ``out``: optional list of float64 [n_rows, N] host tensors
    (pinned for full speed) that receive the results."""
    Bs = list(Bs)
    if not Bs:
        return []
    N = Bs[0].n_cols
    for B in Bs:
        if V.n_cols != B.n_rows or B.n_cols != N:
            raise ValueError(f"dimension mismatch: {V.n_cols} vs {B.n_rows}")
    if V.n_rows == 0 or N == 0:
        return [DenseMatrix(V.n_rows, N, np.zeros((V.n_rows, N))) for _ in Bs]
    pipe = SpmmPipeline(V, N, precision)
    outs = out if out is not None else [pinned_dense(V.n_rows, N) for _ in Bs]
    for k, B in enumerate(Bs):
        src = B if isinstance(B, torch.Tensor) else host_tensor(np.asarray(B.data, dtype=np.float64))
        pipe.step(k, src, outs[k])
    pipe.synchronize()
    pipe.check_finite()
    return [DenseMatrix(V.n_rows, N, o.numpy()) for o in outs]

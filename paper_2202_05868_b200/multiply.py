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

__all__ = ["spmm_vbr", "spmm_vbr_device", "upload_dense"]


def upload_dense(B, precision: str, device=None) -> torch.Tensor:
    """Host float64 [K, N] → device tensor of the kernel dtype with a 16-byte aligned row stride."""
    dev = device or L.require_cuda()
    a = np.ascontiguousarray(np.asarray(B.data if hasattr(B, "data") else B, dtype=np.float64))
    K, N = a.shape
    td = L.PRECISION[precision]
    ld = (N + 7) // 8 * 8
    src = host_tensor(a).to(dev)
    buf = torch.empty((K, ld), dtype=L.TORCH_DTYPE[td], device=dev)
    L.check(L.lib().rb_convert_f64(L.ptr(src), K, N, N, L.ptr(buf), td, ld, L.stream_handle()))
    return buf[:, :N]


def spmm_vbr_device(V, B: torch.Tensor, out=None, precision=None) -> torch.Tensor:
    """Torch-native entry: V (our VbrMatrix or DeviceVbr), B device tensor → fp32 device C."""
    dv = V if hasattr(V, "spmm") else device_vbr_of(V)
    return dv.spmm(B, out=out, precision=precision)


def spmm_vbr(V, B, threads: int = 1, *, precision: str | None = None) -> DenseMatrix:
    """Block-based product with un-permute (multiply.py:72-97); float64 DenseMatrix result."""
    if V.n_cols != B.n_rows:
        raise ValueError(f"dimension mismatch: {V.n_cols} vs {B.n_rows}")
    prec = precision or config.default_precision()
    dv = device_vbr_of(V)
    N = B.n_cols
    if V.n_rows == 0 or N == 0:
        return DenseMatrix(V.n_rows, N, np.zeros((V.n_rows, N)))
    Bd = upload_dense(B, prec)
    C32 = dv.spmm(Bd, precision=prec)
    C64 = torch.empty((V.n_rows, N), dtype=torch.float64, device=C32.device)
    L.check(L.lib().rb_widen_f32(L.ptr(C32), V.n_rows, N, N, L.ptr(C64), N, L.stream_handle()))
    return DenseMatrix(V.n_rows, N, C64.cpu().numpy())

"""ctypes binding of librowblock_b200.so (the C ABI declared in include/rowblock_b200.h).

The product path has no CPU fallback: if the library (or a CUDA device) is
missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ROWBLOCK_B200_LIB") or os.path.join(HERE, "librowblock_b200.so")  # override: experiments

RB_OK, RB_EINVAL, RB_ECUDA, RB_ENOMEM, RB_EUNSUPPORTED = 0, 1, 2, 3, 4
RB_F32, RB_BF16, RB_F16, RB_F64 = 0, 1, 2, 3
RB_JACCARD, RB_COSINE = 0, 1

TORCH_DTYPE = {RB_F32: torch.float32, RB_BF16: torch.bfloat16, RB_F16: torch.float16, RB_F64: torch.float64}
PRECISION = {"bf16": RB_BF16, "fp16": RB_F16, "fp32": RB_F32, "fp64": RB_F64}

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
INT = ctypes.c_int
SZ = ctypes.c_size_t


class VbrDevice(ctypes.Structure):
    """Mirror of ``rb_vbr_device``."""

    _fields_ = [
        ("n_rows", I64), ("n_cols", I64), ("n_block_rows", I64), ("n_blocks", I64), ("n_seg", I64),
        ("total_tile_rows", I64), ("dp", I32), ("tile_dtype", I32),
        ("row_partition", P), ("row_perm", P), ("blk_ptr", P), ("blk_col", P), ("grp_tile_row", P),
        ("col_bounds", P), ("tiles", P), ("cmp_ptr", P), ("cmp_col", P), ("cmp_val", P), ("cmp_h", I32),
    ]


class Sparse24Device(ctypes.Structure):
    """Mirror of ``rb_sparse24_device``."""

    _fields_ = [("sp_tiles", P), ("sp_meta", P), ("sp_tile_row", P), ("total_sp_rows", I64), ("res_ptr", P),
                ("res_col", P), ("res_val", P), ("n_residuals", I64)]


class SpmmInfo(ctypes.Structure):
    _fields_ = [("n_items_tall", I64), ("n_items_short", I64), ("n_items_simt", I64),
                ("executed_flops", ctypes.c_double), ("vbr_flops", ctypes.c_double), ("row_begin_perm", I64),
                ("n_items_skinny", I64), ("n_launches", I64), ("core_vbr_flops", ctypes.c_double),
                ("n_sweep_steps", I64), ("sweep_slots", I64)]


_lib = None


def lib():
    """Load the shared library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(python -m paper_2202_05868_b200._build) first; there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        L.rb_last_error_string.restype = ctypes.c_char_p
        L.rb_abi_version.restype = INT
        L.rb_block_1sa_workspace_size.argtypes = [I64, I64, I64, INT, ctypes.POINTER(SZ)]
        L.rb_block_1sa.argtypes = [I64, I64, I64, P, P, P, I64, ctypes.c_double, INT, INT, INT, INT, P, SZ,
                                   P, P, P, P, P, P, ctypes.POINTER(I64), P]
        L.rb_vbr_workspace_size.argtypes = [I64, I64, I64, ctypes.POINTER(SZ)]
        L.rb_vbr_plan.argtypes = [I64, I64, P, P, P, I64, P, P, I64, P, SZ, P, P, P, P, P,
                                  ctypes.POINTER(I64), ctypes.POINTER(I64), P]
        L.rb_vbr_emit.argtypes = [I64, P, P, P, P, I64, I64, P, SZ, P, P, P, P, P, P, I32, I32, I64, P]
        L.rb_vbr_compact_count.argtypes = [I64, P, P, P, I64, I32, P, ctypes.POINTER(I64), P]
        L.rb_vbr_compact_emit.argtypes = [I64, P, P, P, P, P, I32, P, P, P]
        L.rb_spmm_plan_create.argtypes = [ctypes.POINTER(VbrDevice), I64, I32, I32, I32, ctypes.POINTER(P), P]
        L.rb_spmm_plan_create_ex.argtypes = [ctypes.POINTER(VbrDevice), I64, I32, I32, I32, I32, ctypes.POINTER(P), P]
        L.rb_spmm_plan_info.argtypes = [P, ctypes.POINTER(SpmmInfo)]
        L.rb_spmm_execute.argtypes = [P, P, I64, P, I64, P]
        L.rb_spmm_execute_f64.argtypes = [P, P, I64, P, I64, P]
        L.rb_spmm_execute_fanout.argtypes = [P, P, I64, P, I64, P, I32, P, P]
        L.rb_spmm_plan_destroy.argtypes = [P]
        L.rb_convert_f64.argtypes = [P, I64, I64, I64, P, I32, I64, P]
        L.rb_convert_f64_checked.argtypes = [P, I64, I64, I64, P, I32, I64, P, P]
        L.rb_widen_f32.argtypes = [P, I64, I64, I64, P, I64, P]
        L.rb_group_stats_workspace_size.argtypes = [I64, ctypes.POINTER(SZ)]
        L.rb_group_stats.argtypes = [I64, I64, P, P, P, I64, P, P, P, P, I64, ctypes.c_double, P, SZ, P, P, P, P,
                                     ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I64),
                                     ctypes.POINTER(I64), P]
        L.rb_csr_plan_create.argtypes = [I64, I64, P, I64, I32, ctypes.POINTER(P), P]
        L.rb_csr_execute.argtypes = [P, P, P, P, P, I64, P, I64, P]
        L.rb_csr_plan_destroy.argtypes = [P]
        L.rb_sparse24_layout.argtypes = [ctypes.POINTER(VbrDevice), P, ctypes.POINTER(I64), ctypes.POINTER(I64), P]
        L.rb_sparse24_workspace_size.argtypes = [I64, I64, ctypes.POINTER(SZ)]
        L.rb_sparse24_emit.argtypes = [ctypes.POINTER(VbrDevice), P, P, P, I32, I64, I64, P, SZ, P, P, P, P, P, I64,
                                       ctypes.POINTER(I64), P]
        L.rb_spmm_plan_attach_sparse24.argtypes = [P, ctypes.POINTER(Sparse24Device), P]
        for name in ("rb_sparse24_layout", "rb_sparse24_workspace_size", "rb_sparse24_emit",
                     "rb_spmm_plan_attach_sparse24"):
            getattr(L, name).restype = INT
        for name in ("rb_csr_plan_create", "rb_csr_execute", "rb_csr_plan_destroy"):
            getattr(L, name).restype = INT
        for name in ("rb_block_1sa_workspace_size", "rb_block_1sa", "rb_vbr_workspace_size", "rb_vbr_plan",
                     "rb_vbr_emit", "rb_vbr_compact_count", "rb_vbr_compact_emit", "rb_spmm_plan_create", "rb_spmm_plan_create_ex", "rb_spmm_plan_info", "rb_spmm_execute", "rb_spmm_execute_f64", "rb_spmm_execute_fanout",
                     "rb_spmm_plan_destroy", "rb_convert_f64", "rb_convert_f64_checked", "rb_widen_f32", "rb_group_stats_workspace_size",
                     "rb_group_stats"):
            getattr(L, name).restype = INT
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == RB_OK:
        return
    msg = lib().rb_last_error_string().decode(errors="replace")
    if rc == RB_EINVAL:
        raise ValueError(msg)
    if rc == RB_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"rowblock_b200 error {rc}: {msg}")


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("rowblock_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def ptr(t) -> P:
    return P(0 if t is None else t.data_ptr())


def stream_handle(stream=None) -> P:
    s = stream if stream is not None else torch.cuda.current_stream()
    return P(s.cuda_stream)

"""paper_2202_05868_b200 — B200-native 1-SA → VBR → SpMM (arXiv 2202.05868).

Drop-in for the reference package rowblock v0.1.0 on its hot path:

    block_1sa(A, partition, policy, use_compression=True) -> RowGrouping   (blocking.py:283)
    vbr_from_grouping(A, grouping, partition) -> VbrMatrix                 (vbr.py:88)
    spmm_vbr(V, B, threads=1) -> DenseMatrix                               (multiply.py:72)

with the reference's boundary types (CsrMatrix, DenseMatrix, ColumnPartition,
RowGroup, RowGrouping, MergePolicy, VbrBlock, VbrMatrix).  All compute runs in
hand-written sm_100a CUDA (librowblock_b200.so, C ABI in include/rowblock_b200.h);
there is no CPU fallback.  The torch-native, HBM-resident API is in ``device``.
"""

from .blocking import block_1sa
from .config import default_precision, set_default_precision
from .device import DeviceCsr, DeviceGrouping, DeviceVbr, block_1sa_device
from .metrics import (BlockingCurve, BlockingStats, DensityReport, GroupDensity, blocking_curve, blocking_stats,
                      curve_select, verify_density_bound)
from .multiply import SpmmPipeline, pinned_dense, spmm_csr, spmm_vbr, spmm_vbr_device, spmm_vbr_many
from .types import (ColumnPartition, CsrMatrix, DenseMatrix, MergePolicy, RowGroup, RowGrouping, VbrBlock,
                    VbrMatrix, csr_from_triplets)
from .mtxio import MatrixMarketError, read_matrix_market, read_matrix_market_device, write_matrix_market
from .vbr import load_vbr, save_vbr, vbr_from_grouping, vbr_from_json, vbr_to_json

__all__ = [
    "block_1sa", "vbr_from_grouping", "spmm_vbr", "spmm_vbr_many", "spmm_vbr_device", "block_1sa_device",
    "SpmmPipeline", "pinned_dense", "spmm_csr", "blocking_stats", "blocking_curve", "curve_select",
    "verify_density_bound", "BlockingStats", "BlockingCurve", "GroupDensity", "DensityReport",
    "MatrixMarketError", "read_matrix_market", "read_matrix_market_device", "write_matrix_market", "load_vbr",
    "save_vbr", "vbr_from_json", "vbr_to_json",
    "DeviceCsr", "DeviceGrouping", "DeviceVbr", "ColumnPartition", "CsrMatrix", "DenseMatrix", "MergePolicy",
    "RowGroup", "RowGrouping", "VbrBlock", "VbrMatrix", "csr_from_triplets", "default_precision",
    "set_default_precision",
]
__version__ = "0.1.0"

"""block_1sa — drop-in for rowblock.blocking.block_1sa (blocking.py:283-306) on the GPU.

Same signature, defaults, return type and error behaviour.  The quotient
bitsets, compression, greedy scan and grouping assembly all run on the device
(csrc/blocking.cu through rb_block_1sa); the returned RowGrouping carries the
device arrays in ``.device`` so vbr_from_grouping can reuse them without a
round trip.
"""

from __future__ import annotations

from . import _forkproxy
from .device import DeviceCsr, block_1sa_device
from .types import ColumnPartition, MergePolicy, RowGrouping

__all__ = ["block_1sa", "MergePolicy"]


def block_1sa(A, partition: ColumnPartition, policy: MergePolicy, use_compression: bool = True) -> RowGrouping:
    """Group the rows of A by greedy similarity against the partition (bit-exact with the reference)."""
    if partition.n_cols != A.n_cols:
        raise ValueError("partition inconsistent with matrix dimensions")
    if _forkproxy.in_bad_fork():  # forked pool worker of a CUDA parent: run in a spawned helper
        return _forkproxy.call("block_1sa", A, partition, policy, use_compression)
    dA = DeviceCsr.from_host(A)
    dg = block_1sa_device(dA, partition, policy, use_compression)
    dg.csr = dA
    dg.source = A
    return dg.to_host()

"""vbr_from_grouping — drop-in for rowblock.vbr.vbr_from_grouping (vbr.py:88-125) on the GPU.

The block structure (stored block columns recomputed from the data,
vbr.py:106-112) and the padded dense tiles are built on the device
(csrc/vbr_build.cu through rb_vbr_plan / rb_vbr_emit).  The returned VbrMatrix
has the reference's attributes; its float64 ``block_rows`` payloads are
materialised lazily (also on the device) the first time they are read.
"""

from __future__ import annotations

import numpy as np

from . import config
from .device import DeviceCsr, DeviceVbr
from .types import ColumnPartition, VbrMatrix

__all__ = ["vbr_from_grouping", "VbrMatrix", "vbr_to_json", "vbr_from_json", "save_vbr", "load_vbr"]


def _device_csr_for(A, grouping):
    dg = getattr(grouping, "device", None)
    if dg is not None and getattr(dg, "source", None) is A and getattr(dg, "csr", None) is not None:
        return dg.csr
    return DeviceCsr.from_host(A)


def vbr_from_grouping(A, grouping, partition: ColumnPartition) -> VbrMatrix:
    """Materialise the VBR form of A under the given row grouping (vbr.py:88-125)."""
    if len(grouping.group_of) != A.n_rows or partition.n_cols != A.n_cols:
        raise ValueError("grouping/partition inconsistent with matrix dimensions")
    from . import _forkproxy
    if _forkproxy.in_bad_fork():  # forked pool worker of a CUDA parent: run in a spawned helper
        return _forkproxy.call("vbr_from_grouping", A, grouping, partition)
    dA = _device_csr_for(A, grouping)
    dg = getattr(grouping, "device", None)
    if dg is not None and dg.n_rows == A.n_rows:
        row_perm = dg.row_perm
        row_partition = dg.group_ptr[: dg.n_groups + 1]
        rp_host = row_partition.cpu().numpy()
        perm_host = None
    else:
        groups = grouping.groups
        perm_host = np.concatenate([np.asarray(g.rows, np.int64) for g in groups]) if groups else np.zeros(0, np.int64)
        rp_host = np.zeros(len(groups) + 1, np.int64)
        np.cumsum([len(g.rows) for g in groups], out=rp_host[1:])
        row_perm, row_partition = perm_host, rp_host
    dv = DeviceVbr.build(dA, partition, row_perm, row_partition, dtypes=(config.default_precision(),))
    if perm_host is None:
        perm_host = dv.row_perm64.cpu().numpy()
    return VbrMatrix(A.n_rows, A.n_cols, rp_host, partition, perm_host, device=dv)


def device_vbr_of(V) -> DeviceVbr:
    """The device form of any VbrMatrix (ours: cached; a host-only one, e.g. the reference's or one
    read from JSON: rebuilt on the device from its payload nonzeros)."""
    dv = getattr(V, "device", None)
    if isinstance(dv, DeviceVbr):
        return dv
    from .types import CsrMatrix
    bounds = np.asarray(V.col_partition.boundaries, np.int64)
    rows, cols, vals = [], [], []
    rp = np.asarray(V.row_partition, np.int64)
    perm = np.asarray(V.row_perm, np.int64)
    for g, br in enumerate(V.block_rows):
        orig = perm[rp[g]:rp[g + 1]]
        for blk in br:
            r, c = np.nonzero(blk.data)
            rows.append(orig[r])
            cols.append(c + bounds[blk.bcol])
            vals.append(blk.data[r, c])
    from .types import csr_from_coo
    if rows:
        A = csr_from_coo(V.n_rows, V.n_cols, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))
    else:
        A = CsrMatrix(V.n_rows, V.n_cols, np.zeros(V.n_rows + 1, np.int64), [], [])
    dv = DeviceVbr.build(DeviceCsr.from_host(A), V.col_partition, perm, rp, dtypes=())
    try:
        V.device = dv
    except Exception:  # frozen reference dataclass: no caching
        pass
    return dv


# ------------------------------------------------------------------------------------------ JSON
# Debug interchange, same document as the reference (vbr.py:167-202): payloads as flat lists.


def vbr_to_json(V) -> dict:
    return {
        "n_rows": V.n_rows,
        "n_cols": V.n_cols,
        "row_partition": np.asarray(V.row_partition).tolist(),
        "col_boundaries": np.asarray(V.col_partition.boundaries).tolist(),
        "row_perm": np.asarray(V.row_perm).tolist(),
        "blocks": [{"brow": g, "bcol": int(b.bcol), "data": b.data.ravel().tolist()}
                   for g in range(V.n_block_rows) for b in V.block_rows[g]],
    }


def vbr_from_json(doc: dict) -> VbrMatrix:
    from .types import VbrBlock

    part = ColumnPartition(doc["col_boundaries"][-1], np.asarray(doc["col_boundaries"]))
    row_partition = np.asarray(doc["row_partition"], dtype=np.int64)
    widths = part.widths
    block_rows = [[] for _ in range(len(row_partition) - 1)]
    for b in doc["blocks"]:
        g, bcol = b["brow"], b["bcol"]
        h = int(row_partition[g + 1] - row_partition[g])
        block_rows[g].append(VbrBlock(bcol, np.asarray(b["data"], dtype=np.float64).reshape(h, widths[bcol])))
    return VbrMatrix(doc["n_rows"], doc["n_cols"], row_partition, part, np.asarray(doc["row_perm"]), block_rows)


def save_vbr(path, V) -> None:
    import json

    with open(path, "w", encoding="ascii") as fh:
        json.dump(vbr_to_json(V), fh)


def load_vbr(path) -> VbrMatrix:
    import json

    with open(path, "r", encoding="ascii") as fh:
        return vbr_from_json(json.load(fh))

"""Fused all-gather of C (rb_spmm_execute_fanout, dist.FusedGather).

The epilogues store every C element into the caller's C and, at the same offset, into each peer
buffer.  On a multi-GPU box the peers are the other ranks' symmetric-memory C mapped over NVLink;
the kernel code does not know the difference, so here the "peers" are plain buffers on one GPU and
every rank's kernel runs in turn (no kernel waits on another).  Bars:
  * fan-out copies are bit-identical to the plain rb_spmm_execute product (same plan, same kernels);
  * W ranks' sub-VBRs (dist.shard_vbr) writing their rows at their global source rows (c_rows) into
    all W buffers leave the whole product, in source row order, in every buffer — what NCCL
    all-gather + un-permute (dist.gather_c, multiply.py:90) produces — within the fp32
    reassociation tolerance of the sharded plans (1e-5 of max|C|), and the W buffers bit-identical.
"""
import numpy as np
import pytest
import torch

import paper_2202_05868_b200 as rb
from conftest import golden_b, load_golden
from test_gpu_parity import csr_of, part_of, policy_of

pytestmark = pytest.mark.gpu

CASES = [("cfg5_s32", "bf16", "0"), ("cfg5_s32", "bf16", "2"), ("cfg4_s8", "bf16", "0"), ("rmat12_t3", "bf16", "0"),
         ("rmat12_t3", "fp32", "0"), ("cfg2b_s16", "bf16", "0"), ("small", "fp32", "0")]


def _vbr(name):
    case = load_golden(name) if name != "small" else None
    if case is None:  # a few rows without nonzeros (zero-row kernel) and an fp32 SIMT block row
        rng = np.random.default_rng(3)
        d = (rng.random((300, 500)) < 0.05) * rng.standard_normal((300, 500))
        d[rng.random(300) < 0.2] = 0.0
        d[:40, :64] = rng.standard_normal((40, 64))
        import scipy.sparse as sp

        m = sp.csr_matrix(d)
        A = rb.CsrMatrix(300, 500, m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data)
        q = rb.ColumnPartition.uniform(500, 64)
        V = rb.vbr_from_grouping(A, rb.block_1sa(A, q, rb.MergePolicy(tau=0.5), True), q)
        return A, q, V, rng.standard_normal((500, 96))
    A, q = csr_of(case), part_of(case)
    V = rb.vbr_from_grouping(A, rb.block_1sa(A, q, policy_of(case), True), q)
    B = golden_b(case)
    if B is None:  # fixtures recorded without B (structure-only cases)
        B = np.random.default_rng(5).standard_normal((A.n_cols, 192))
    return A, q, V, B


@pytest.mark.parametrize("name,precision,sweep", CASES)
def test_fanout_copies_equal_plain_product(name, precision, sweep, monkeypatch):
    monkeypatch.setenv("RB_SWEEP", sweep)
    A, q, V, Bh = _vbr(name)
    tdt = {"bf16": torch.bfloat16, "fp32": torch.float32}[precision]
    B = torch.from_numpy(Bh).to(tdt).cuda()
    plain = V.device.spmm(B, precision=precision)
    bufs = [torch.full_like(plain, float("nan")) for _ in range(4)]
    V.device.spmm_fanout(B, bufs[0], bufs[1:], precision=precision)
    torch.cuda.synchronize()
    for i, t in enumerate(bufs):
        assert torch.equal(t, plain), (name, precision, sweep, i)


@pytest.mark.parametrize("name", ["cfg5_s32", "cfg4_s8", "rmat12_t3"])
def test_fanout_shards_assemble_full_product_in_every_buffer(name):
    from paper_2202_05868_b200 import dist as rbdist
    from paper_2202_05868_b200.device import DeviceCsr, block_1sa_device
    from paper_2202_05868_b200.types import MergePolicy

    case = load_golden(name)
    A, q = csr_of(case), part_of(case)
    dA = DeviceCsr.from_host(A)
    dg = block_1sa_device(dA, q, MergePolicy(tau=float(case["tau"])), True)
    B = torch.from_numpy(golden_b(case)).to(torch.bfloat16).cuda()
    full = rb.vbr_from_grouping(A, rb.block_1sa(A, q, policy_of(case), True), q).device.spmm(B, precision="bf16")
    for world in (2, 3, 8):
        bufs = [torch.full_like(full, float("nan")) for _ in range(world)]
        for k in range(world):
            dv, (b, e), _ = rbdist.shard_vbr(dA, q, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], "bf16", k, world)
            assert torch.equal(dv.global_rows.cpu(), rbdist.global_rows_of(dg.row_perm[: A.n_rows].cpu(), b, e))
            if e > b:
                dv.spmm_fanout(B, bufs[k], [bufs[j] for j in range(world) if j != k], c_rows=dv.global_rows,
                               precision="bf16")
        torch.cuda.synchronize()
        for j in range(world):
            assert not torch.isnan(bufs[j]).any(), (name, world, j)
            assert torch.equal(bufs[j], bufs[0]), (name, world, j)
        err = (bufs[0].double() - full.double()).abs().max().item()
        assert err <= 1e-5 * max(1.0, full.abs().max().item()), (name, world, err)


def test_fanout_argument_checks():
    from paper_2202_05868_b200 import _lib as L

    A, q, V, Bh = _vbr("cfg5_s32")
    B = torch.from_numpy(Bh).to(torch.bfloat16).cuda()
    out = torch.empty((A.n_rows, B.shape[1]), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        V.device.spmm_fanout(B, out, [torch.empty_like(out) for _ in range(8)])
    with pytest.raises(ValueError):
        V.device.spmm_fanout(B, out, [torch.empty_like(out, dtype=torch.float64)])
    with pytest.raises(ValueError):
        V.device.spmm_fanout(B, out, [], c_rows=torch.zeros(3, dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        V.device.spmm_fanout(B, out, [], c_rows=torch.full((A.n_rows,), A.n_rows, dtype=torch.int32, device="cuda"))
    # the C ABI refuses misaligned fan-out buffers and more than 7 peers
    h = V.device.plan(B.shape[1], "bf16")
    flat = torch.empty(A.n_rows * B.shape[1] + 1, dtype=torch.float32, device="cuda")
    import ctypes
    bad = (ctypes.c_void_p * 1)(flat.data_ptr() + 4)
    rc = L.lib().rb_spmm_execute_fanout(h, L.ptr(B), B.stride(0), L.ptr(out), out.stride(0), bad, 1, None,
                                        L.stream_handle())
    assert rc != 0
    many = (ctypes.c_void_p * 8)(*([out.data_ptr()] * 8))
    rc = L.lib().rb_spmm_execute_fanout(h, L.ptr(B), B.stride(0), L.ptr(out), out.stride(0), many, 8, None,
                                        L.stream_handle())
    assert rc != 0


@pytest.mark.timeout(300)
def test_fused_gather_symmetric_memory_world1():
    """dist.FusedGather's plumbing on a real device: NCCL process group, torch symmetric-memory C,
    rendezvous and the device barrier, at world size 1 (no peers; one GPU is all this pod has).
    The gathered C must equal the plain product bit for bit."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2202_05868_b200 import dist as rbdist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        A, q, V, Bh = _vbr("cfg5_s32")
        B = torch.from_numpy(Bh).to(torch.bfloat16).cuda()
        plain = V.device.spmm(B, precision="bf16")
        try:
            fg = rbdist.FusedGather(A.n_rows, B.shape[1], torch.device("cuda:0"))
        except Exception as exc:  # noqa: BLE001
            pytest.skip(f"torch symmetric memory unavailable here: {type(exc).__name__}: {exc}")
        assert fg.peers == []
        C = fg.run(V.device, B, precision="bf16")
        torch.cuda.synchronize()
        assert torch.equal(C, plain)
    finally:
        dist.destroy_process_group()

"""World-size-2 gloo test of the sharded SpMM host logic (bench.py --gpus N path).

Each rank takes its shard of the permuted rows from the same planner the GPU plan uses
(rb_spmm_shard_range), computes its C rows with the CPU oracle, and the ranks all-gather +
un-permute with paper_2202_05868_b200.dist.gather_c.  The gathered C must equal the
single-process oracle C exactly (disjoint rows, no reduction across ranks)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, golden_b, load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from conftest import golden_b as gb, load_golden as lg
        from paper_2202_05868_b200 import dist as rbdist

        case = lg(name)
        B = gb(case)
        rp, bp = case["row_partition"], case["blk_ptr"]
        ranges = rbdist.all_ranges(rp, bp, "bf16", 64, world)
        b, e = ranges[rank]
        pay = oracle.vbr_payloads(case["row_ptr"], case["col_idx"], case["values"], case["boundaries"],
                                  case["row_perm"], rp, bp, case["blk_col"])
        # this rank's block rows only (cuts fall on M-tile starts: split a tall block row by rows)
        C_perm = np.zeros((e - b, B.shape[1]))
        bounds = case["boundaries"]
        for g in range(len(rp) - 1):
            lo, hi = int(rp[g]), int(rp[g + 1])
            a, z = max(lo, b), min(hi, e)
            if a >= z:
                continue
            acc = np.zeros((z - a, B.shape[1]))
            for s, data in pay[g]:
                acc += data[a - lo:z - lo] @ B[bounds[s]:bounds[s + 1]]
            C_perm[a - b:z - b] = acc
        full = rbdist.gather_c(torch.from_numpy(C_perm), torch.from_numpy(case["row_perm"]), ranges)
        if rank == 0:
            q.put(full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg1_full", "cfg5_s32"])
def test_two_rank_sharded_spmm_gather_matches_single_process(name):
    import oracle

    case = load_golden(name)
    B = golden_b(case)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pay = oracle.vbr_payloads(case["row_ptr"], case["col_idx"], case["values"], case["boundaries"], case["row_perm"],
                              case["row_partition"], case["blk_ptr"], case["blk_col"])
    ref = oracle.spmm_vbr_np(pay, case["row_perm"], case["row_partition"], case["boundaries"], B)
    np.testing.assert_allclose(full, ref, rtol=1e-12, atol=1e-12)
    r = np.random.default_rng(7).standard_normal(B.shape[1])
    np.testing.assert_allclose(full @ r, case["C_dot_r"], rtol=1e-9, atol=1e-9)


def _worker_subvbr(rank, world, port, name, q):
    """bench.py --gpus N's per-rank path: the shard's rows become a sub-matrix (dist.take_rows) with
    its own grouping (dist.shard_grouping: identity row order, cuts at the global block rows), the
    rank multiplies only that sub-VBR (here: the oracle on its payloads) and gather_c assembles C."""
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from conftest import golden_b as gb, load_golden as lg
        from paper_2202_05868_b200 import dist as rbdist
        from paper_2202_05868_b200.device import DeviceCsr

        case = lg(name)
        B = gb(case)
        rp, bp = case["row_partition"], case["blk_ptr"]
        ranges = rbdist.all_ranges(rp, bp, "bf16", 64, world)
        b, e = ranges[rank]
        rows, cuts = rbdist.shard_grouping(case["row_perm"], rp, b, e)
        A = DeviceCsr(int(case["n_rows"]), int(case["n_cols"]), torch.from_numpy(case["row_ptr"]),
                      torch.from_numpy(case["col_idx"]), torch.from_numpy(case["values"]))
        sub = rbdist.take_rows(A, rows)
        srp, sci, sval = sub.row_ptr.numpy(), sub.col_idx.numpy(), sub.values.numpy()
        ident = np.arange(e - b, dtype=np.int64)
        cuts = cuts.numpy()
        sbp, sbc = oracle.vbr_blocks(srp, sci, case["boundaries"], ident, cuts)
        pay = oracle.vbr_payloads(srp, sci, sval, case["boundaries"], ident, cuts, sbp, sbc)
        C_local = oracle.spmm_vbr_np(pay, ident, cuts, case["boundaries"], B)  # permuted order = local order
        full = rbdist.gather_c(torch.from_numpy(C_local), torch.from_numpy(case["row_perm"]), ranges)
        # the fused gather's row map: the rank stores its rows at global_rows_of (= dv.global_rows,
        # rb_spmm_execute_fanout's c_rows) in every rank's full C; disjoint rows, so summing the
        # ranks' stores must give exactly the NCCL gather + un-permute result
        fan = torch.zeros_like(full)
        fan[rbdist.global_rows_of(case["row_perm"], b, e).to(torch.int64)] = torch.from_numpy(C_local)
        dist.all_reduce(fan)
        if rank == 0:
            q.put(full.numpy())
            q.put(fan.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("cfg1_full", 2), ("cfg5_s32", 2), ("cfg4_s8", 3)])
def test_sharded_sub_vbr_gather_matches_single_process(name, world):
    import oracle

    case = load_golden(name)
    B = golden_b(case)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_subvbr, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=300)
    fan = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pay = oracle.vbr_payloads(case["row_ptr"], case["col_idx"], case["values"], case["boundaries"], case["row_perm"],
                              case["row_partition"], case["blk_ptr"], case["blk_col"])
    ref = oracle.spmm_vbr_np(pay, case["row_perm"], case["row_partition"], case["boundaries"], B)
    np.testing.assert_allclose(full, ref, rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(fan, full)  # fused-gather row map == gather_c + un-permute

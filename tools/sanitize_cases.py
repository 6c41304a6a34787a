"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
1-SA (dense and sparse greedy kernels), VBR build, and every SpMM kernel family on reference-made
golden inputs: fp32 check path (cfg1), short swap-AB + sweep (cfg5_s32), tall with a forced split-K
tail (cfg4_s8), skinny with split hub rows (rmat12), 8-shard plans, CSR comparator.  Each product is
compared with the golden checksums so a sanitizer run also proves the results.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import paper_2202_05868_b200 as rb  # noqa: E402
from conftest import golden_b, load_golden  # noqa: E402


def case_objs(name):
    c = load_golden(name)
    A = rb.CsrMatrix(int(c["n_rows"]), int(c["n_cols"]), c["row_ptr"], c["col_idx"], c["values"])
    q = rb.ColumnPartition(int(c["n_cols"]), c["boundaries"])
    pol = rb.MergePolicy(tau=float(c["tau"]))
    return c, A, q, pol


def check(name, C, c, tol):
    B = golden_b(c)
    r = np.random.default_rng(7).standard_normal(B.shape[1])
    dev = np.abs(C @ r - c["C_dot_r"]).max()
    scale = np.abs(c["C_dot_r"]).max() + 1.0
    assert dev <= tol * scale * 10, (name, dev, scale)
    print(f"{name}: ok (max |C·r - ref| = {dev:.3e})", flush=True)


def main():
    only = sys.argv[1:]
    runs = [("cfg1_full", "fp32", {}), ("cfg1_full", "bf16", {}), ("cfg5_s32", "bf16", {}),
            ("cfg5_s32", "bf16", {"RB_SWEEP": "2"}), ("cfg4_s8", "bf16", {"RB_TALL_SPLIT": "4"}),
            ("rmat12_t3", "bf16", {"RB_SKINNY_PART_MAX": "8"}), ("rmat12_t9", "fp32", {})]
    for name, prec, env in runs:
        if only and name not in only:
            continue
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            c, A, q, pol = case_objs(name)
            g = rb.block_1sa(A, q, pol)
            assert np.array_equal(g.group_of, c["group_of"]), name
            V = rb.vbr_from_grouping(A, g, q)
            B = golden_b(c)
            C = rb.spmm_vbr(V, rb.DenseMatrix.from_array(B), precision=prec).data
            check(f"{name} {prec} {env}", C, c, 1e-5 if prec == "fp32" else 1e-2)
            if name == "rmat12_t3":  # 8-shard plans and the CSR comparator on the same input
                import torch
                dv = V.device
                Bd = torch.from_numpy(B).to(torch.bfloat16).cuda()
                full = dv.spmm(Bd, precision="bf16")
                out = torch.full_like(full, float("nan"))
                for k in range(8):
                    dv.spmm(Bd, out=out, precision="bf16", shard=k, n_shards=8)
                torch.cuda.synchronize()
                assert not torch.isnan(out).any()
                Cc = rb.spmm_csr(A, rb.DenseMatrix.from_array(B), precision="bf16").data
                check(f"{name} csr", Cc, c, 1e-2)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    # sparse (large-W) greedy 1-SA path on the R-MAT goldens
    os.environ["RB_1SA_MODE"] = "sparse"
    for name in ("rmat12_t3", "rmat12_t9"):
        if only and name not in only:
            continue
        c, A, q, pol = case_objs(name)
        g = rb.block_1sa(A, q, pol)
        assert np.array_equal(g.group_of, c["group_of"]), name
        print(f"{name}: sparse 1-SA ok", flush=True)


if __name__ == "__main__":
    main()

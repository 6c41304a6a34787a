"""Command-line front end on the GPU path — the reference's ``rowblock block`` / ``rowblock bench``
(cli.py:244-349) with B200 kernels and GPU columns.

    python -m paper_2202_05868_b200.cli block in.mtx --dw 64 --tau 0.7 [--out grouping.json]
    python -m paper_2202_05868_b200.cli bench in.mtx --dw 32 64 --tau 0.7 -N 128 512 [--runs 3]

``block`` prints the reference's summary line and writes the same grouping JSON
(docs/formats.md "Grouping JSON").  ``bench`` writes bench.csv with the reference's
BENCH_COLUMNS (cli.py:39-42) followed by GPU columns; kernel ``csr`` is the CSR gather kernel
(spmm_csr, csrc/csr.cu) and ``vbr`` the VBR path (spmm_vbr: tcgen05 / skinny kernels), both on
device-resident A and B, timed with CUDA events.  As in the reference (cli.py:331-334) the two
kernels' outputs are compared before any timing and a mismatch is a RuntimeError (exit 1); the
tolerance is the fp32-accumulation bound of the chosen precision instead of 1e-9.  The cost-model
columns (tcu_*, multiply.py tcu_cost*) are outside the ported hot path and stay empty.
Exit codes: 0 success, 1 runtime failure, 2 usage error (cli.py:418-427).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np

__all__ = ["BENCH_COLUMNS", "GPU_COLUMNS", "main", "build_parser"]

BENCH_COLUMNS = [
    "matrix", "dw", "tau", "kernel", "threads", "n_dense", "runs",
    "median_s", "mean_s", "tcu_blocked", "tcu_trivial",
]
GPU_COLUMNS = ["precision", "device", "gflops_useful", "n_groups", "n_stored_blocks", "rho_prime"]


def _fmt(v) -> str:
    if v is None:
        return ""
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, float):
        return repr(v)
    return str(v)


def _write_csv(path, columns, rows) -> None:
    with open(path, "w", encoding="ascii") as fh:
        fh.write(",".join(columns) + "\n")
        for row in rows:
            fh.write(",".join(_fmt(row.get(c)) for c in columns) + "\n")


def _out_dir(arg):
    d = Path(arg or os.environ.get("ROWBLOCK_OUT", "."))
    d.mkdir(parents=True, exist_ok=True)
    return d


def _policy_from_flags(args):
    from .types import MergePolicy

    kind = getattr(args, "policy", "bounded")
    sim = getattr(args, "similarity", None)
    if kind == "bounded":
        return MergePolicy(similarity=sim or "jaccard", tau=args.tau, bounded=True, pattern_update=True)
    if kind == "plain":
        return MergePolicy(similarity=sim or "jaccard", tau=args.tau, bounded=False, pattern_update=True)
    raise ValueError(f"unknown policy {kind!r}")


def _load(args):
    from .device import DeviceCsr
    from .mtxio import read_matrix_market

    A = read_matrix_market(args.input)
    if args.scramble_seed is not None:
        raise ValueError("--scramble-seed needs the reference's generators (out of scope here); "
                         "scramble the .mtx file instead")
    return A, DeviceCsr.from_host(A)


def cmd_block(args) -> int:
    from .device import block_1sa_device
    from .metrics import blocking_stats
    from .types import ColumnPartition

    A, dA = _load(args)
    policy = _policy_from_flags(args)
    part = ColumnPartition.uniform(A.n_cols, args.dw)
    dg = block_1sa_device(dA, part, policy, use_compression=not args.no_compress)
    stats = blocking_stats(dA, dg, part, tau=args.tau, check_bound=policy.bounded)
    if args.out:
        g = dg.to_host()
        doc = {"n_rows": A.n_rows, "group_of": g.group_of.tolist(),
               "groups": [{"rows": gr.rows.tolist(), "pattern": gr.pattern.tolist(), "seed_size": gr.seed_size}
                          for gr in g.groups]}
        with open(args.out, "w", encoding="ascii") as fh:
            json.dump(doc, fh)
    print(f"groups={stats.n_groups} stored_blocks={stats.n_stored_blocks} "
          f"rho_prime={stats.rho_prime:.6g} delta_h_prime={stats.delta_h_prime:.6g} "
          f"fill_in={stats.fill_in} density_bound_ok={_fmt(stats.density_bound_ok)}")
    return 0


def _time_device(fn, runs: int):
    import torch

    times = []
    for _ in range(runs):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) * 1e-3)
    return statistics.median(times), statistics.fmean(times)


def cmd_bench(args) -> int:
    import torch

    from .device import DeviceVbr, block_1sa_device
    from .metrics import blocking_stats
    from .multiply import upload_dense
    from .types import ColumnPartition

    A, dA = _load(args)
    policy = _policy_from_flags(args)
    prec = args.precision
    rng = np.random.default_rng(args.dense_seed)
    rows = []
    name = Path(args.input).name
    dev_name = torch.cuda.get_device_name()
    for dw in args.dw:
        part = ColumnPartition.uniform(A.n_cols, dw)
        dg = block_1sa_device(dA, part, policy)
        dv = DeviceVbr.build(dA, part, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=(prec,))
        st = blocking_stats(dA, dg, part)
        for n_dense in args.n_dense:
            B = upload_dense(rng.random((A.n_cols, n_dense)), prec)
            C_csr = dA.spmm(B, precision=prec)
            C_vbr = dv.spmm(B, precision=prec)
            torch.cuda.synchronize()
            err = float((C_csr - C_vbr).abs().max().item()) if A.n_rows else 0.0
            scale = max(1.0, float(C_csr.abs().max().item()) if A.n_rows else 0.0)
            tol = (1e-5 if prec == "fp32" else 1e-4) * scale
            if err > tol:
                raise RuntimeError(f"kernel mismatch before timing: max err {err}")
            for kernel, fn in (("csr", lambda: dA.spmm(B, out=C_csr, precision=prec)),
                               ("vbr", lambda: dv.spmm(B, out=C_vbr, precision=prec))):
                fn()
                med, mean = _time_device(fn, args.runs)
                rows.append({
                    "matrix": name, "dw": dw, "tau": args.tau, "kernel": kernel, "threads": args.threads,
                    "n_dense": n_dense, "runs": args.runs, "median_s": med, "mean_s": mean,
                    "tcu_blocked": None, "tcu_trivial": None, "precision": prec, "device": dev_name,
                    "gflops_useful": 2.0 * A.nnz * n_dense / med / 1e9 if med > 0 else None,
                    "n_groups": st.n_groups, "n_stored_blocks": st.n_stored_blocks, "rho_prime": st.rho_prime,
                })
    out = Path(args.out) if args.out else _out_dir(None) / "bench.csv"
    _write_csv(out, BENCH_COLUMNS + GPU_COLUMNS, rows)
    print(f"wrote {out} ({len(rows)} rows)")
    return 0


def _tau_type(text: str) -> float:
    value = float(text)
    if value < 0.0 or value > 1.0:
        raise argparse.ArgumentTypeError(f"tau must be in [0, 1], got {text}")
    return value


# (flags, keyword arguments) per command; the reference's flag names and defaults, plus --precision
_COMMON = [
    (("input",), {}),
    (("--tau",), dict(type=_tau_type, required=True)),
    (("--policy",), dict(choices=["bounded", "plain"], default="bounded")),
    (("--similarity",), dict(choices=["jaccard", "cosine"])),
    (("--scramble-seed",), dict(type=int)),
]
_COMMANDS = {
    "block": ("group the rows of an .mtx file (device 1-SA)", [
        (("--dw",), dict(type=int, required=True, help="column partition width")),
        (("--no-compress",), dict(action="store_true")),
        (("--out",), dict(help="write the grouping as JSON")),
    ]),
    "bench": ("time the CSR and VBR kernels on the GPU", [
        (("--dw",), dict(type=int, nargs="+", required=True)),
        (("-N", "--n-dense"), dict(type=int, nargs="+", required=True)),
        (("--threads",), dict(type=int, default=1, help="accepted for compatibility (GPU kernels)")),
        (("--runs",), dict(type=int, default=3)),
        (("--dense-seed",), dict(type=int, default=0)),
        (("--precision",), dict(choices=["bf16", "fp16", "fp32"], default="bf16")),
        (("--out",), {}),
    ]),
}


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="rowblock-b200", description="Row blocking + VBR SpMM on B200: block, bench.")
    sub = parser.add_subparsers(dest="command", required=True)
    for name, (help_text, specific) in _COMMANDS.items():
        cmd = sub.add_parser(name, help=help_text)
        for flags, kw in _COMMON + specific:
            cmd.add_argument(*flags, **kw)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    handlers = {"block": cmd_block, "bench": cmd_bench}
    try:
        return handlers[args.command](args)
    except (ValueError, OSError, RuntimeError, KeyError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())

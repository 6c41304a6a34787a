"""Pinned synthetic inputs for the five BASELINE.json configurations.

All random draws use numpy PCG64 (``np.random.default_rng(seed)``, as the
reference's generators do, generators.py:1-6); only the large sorts run in torch
(on the GPU when one is present) — sorting unique keys is deterministic, so the
matrices are identical on every machine.  A values are U[0.1, 1) (the
reference's test convention, conftest.py:12) and are rounded to the kernel
dtype before either path sees them, so the CPU reference (float64 on the
rounded values) and the GPU differ only by fp32 accumulation.

    cfg 1  2048 x 2048, exactly 41,943 nnz uniform,            Δ=64,  τ=0.7, B 2048 x 256  fp32
    cfg 2  32768^2, 64^2 blocks θ=5% ρ=1, +10% uniform noise draws (dedup), rows AND columns
           permuted (literal reading),                       Δ=64,  τ=0.7, B 32768 x 512 bf16
    cfg 2b same, rows-only scramble (stress case)
    cfg 3  R-MAT 2^20, 16 draws/node, (.57,.19,.19,.05), rows scrambled, Δ=32, τ∈{.3..9}, N=128
    cfg 4  4096 x 16384, exactly 10% uniform,                   Δ=128, τ=0.7, B 16384 x 2048 bf16
    cfg 5  262144^2, 64^2 blocks θ=1% ρ=1, rows scrambled,     Δ=64,  τ=0.7, B 262144 x 1024 bf16

``scale`` shrinks the linear dimensions (tests / quick runs); the bench uses scale=1.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .device import DeviceCsr


@dataclass(frozen=True)
class Config:
    name: str
    n_rows: int
    n_cols: int
    delta: int
    tau: float
    N: int
    precision: str
    description: str


CONFIGS = {
    "1": Config("1", 2048, 2048, 64, 0.7, 256, "fp32", "uniform 2048x2048 1%, D=64, tau=0.7, B fp32 N=256"),
    "2": Config("2", 32768, 32768, 64, 0.7, 512, "bf16",
                "hidden-block 32768^2 (64^2 blocks, 5% block density, rows+cols permuted, +10% noise), D=64, N=512"),
    "2b": Config("2b", 32768, 32768, 64, 0.7, 512, "bf16", "config 2 with rows-only scramble (stress)"),
    "3": Config("3", 1 << 20, 1 << 20, 32, 0.7, 128, "bf16", "R-MAT 2^20 deg 16, rows scrambled, D=32, N=128"),
    "4": Config("4", 4096, 16384, 128, 0.7, 2048, "bf16", "DNN layer 4096x16384 90% sparse, D=128, B 16384x2048"),
    "5": Config("5", 262144, 262144, 64, 0.7, 1024, "bf16",
                "hidden-block 262144^2 (64^2 blocks, 1% block density), rows scrambled, D=64, N=1024"),
}

SEEDS = {"1": 1, "2": 2, "2b": 2, "3": 3, "4": 4, "5": 5}


def _round_half_up(x: float) -> int:
    return int(np.floor(x + 0.5))


def _dev(device):
    if device is not None:
        return torch.device(device)
    return torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")


def round_to(x: np.ndarray, precision: str) -> np.ndarray:
    """Correctly rounded float64 -> precision -> float64 (matches the device's __double2bfloat16)."""
    x = np.asarray(x, np.float64)
    if precision == "fp32":
        return x.astype(np.float32).astype(np.float64)
    if precision == "fp16":
        return x.astype(np.float16).astype(np.float64)
    b = np.ascontiguousarray(x).view(np.uint64)
    lsb = (b >> np.uint64(45)) & np.uint64(1)
    return ((b + np.uint64((1 << 44) - 1) + lsb) & ~np.uint64((1 << 45) - 1)).view(np.float64)


def _csr_from_keys(keys: torch.Tensor, n_rows: int, n_cols: int, vals: np.ndarray, dev) -> DeviceCsr:
    """keys = row * n_cols + col, unique (any order) -> DeviceCsr with values assigned in key order."""
    keys, _ = torch.sort(keys)
    rows = torch.div(keys, n_cols, rounding_mode="floor")
    cols = keys - rows * n_cols
    counts = torch.bincount(rows, minlength=n_rows)
    row_ptr = torch.zeros(n_rows + 1, dtype=torch.int64, device=dev)
    row_ptr[1:] = torch.cumsum(counts, 0)
    v = torch.from_numpy(vals).to(dev)
    return DeviceCsr(n_rows, n_cols, row_ptr, cols.contiguous(), v)


def _values(rng, nnz: int, precision: str) -> np.ndarray:
    return round_to(rng.uniform(0.1, 1.0, nnz), precision)


def _blocked_keys(rng, n: int, d: int, theta: float, dev) -> torch.Tensor:
    """Keys of round(theta * #blocks) distinct d x d blocks, every cell filled (rho = 1)."""
    bc = n // d
    n_sel = _round_half_up(theta * bc * bc)
    blocks = np.sort(rng.choice(bc * bc, size=n_sel, replace=False))
    b = torch.from_numpy(blocks).to(dev)
    br = torch.div(b, bc, rounding_mode="floor")
    bcc = b - br * bc
    cell = torch.arange(d * d, device=dev)
    r = (br[:, None] * d + torch.div(cell, d, rounding_mode="floor")[None, :]).reshape(-1)
    c = (bcc[:, None] * d + (cell % d)[None, :]).reshape(-1)
    return r * n + c


def make(name: str, scale: int = 1, device=None, precision: str | None = None):
    """Build config ``name`` → (DeviceCsr, partition boundaries np.int64, Config, meta dict)."""
    cfg = CONFIGS[name]
    dev = _dev(device)
    prec = precision or cfg.precision
    rng = np.random.default_rng(SEEDS[name])
    n_rows, n_cols = cfg.n_rows // scale, cfg.n_cols // scale
    meta = {}
    if name == "1":
        nnz = _round_half_up(0.01 * n_rows * n_cols)
        keys = torch.from_numpy(rng.choice(n_rows * n_cols, size=nnz, replace=False)).to(dev)
        A = _csr_from_keys(keys, n_rows, n_cols, _values(rng, nnz, prec), dev)
    elif name in ("2", "2b", "5"):
        theta = 0.05 if name != "5" else 0.01
        n = n_rows
        keys = _blocked_keys(rng, n, 64, theta, dev)
        meta["planted_nnz"] = int(keys.numel())
        if name != "5":
            n_noise = _round_half_up(0.10 * keys.numel())
            noise = torch.from_numpy(rng.integers(0, n * n, size=n_noise, dtype=np.int64)).to(dev)
            keys = torch.unique(torch.cat([keys, noise]))
        perm_r = torch.from_numpy(rng.permutation(n)).to(dev)
        rows = torch.div(keys, n, rounding_mode="floor")
        cols = keys - rows * n
        if name == "2":
            perm_c = torch.from_numpy(rng.permutation(n)).to(dev)
            cols = perm_c[cols]
        # row scramble: output row i = input row perm[i]  (generators.py:137-145) -> input row r
        # lands at position inv[r]
        inv = torch.empty_like(perm_r)
        inv[perm_r] = torch.arange(n, device=dev)
        keys = inv[rows] * n + cols
        del rows, cols
        A = _csr_from_keys(keys, n, n, _values(rng, int(keys.numel()), prec), dev)
    elif name == "3":
        log2 = int(np.log2(n_rows))
        n = 1 << log2
        draws = n * 16
        cum = np.array([0.57, 0.76, 0.95])
        rows = np.zeros(draws, np.int64)
        cols = np.zeros(draws, np.int64)
        for _ in range(log2):  # generators.py:109-124
            quad = np.searchsorted(cum, rng.random(draws), side="right")
            rows = (rows << 1) | (quad >> 1)
            cols = (cols << 1) | (quad & 1)
        keys = torch.unique(torch.from_numpy(rows * n + cols).to(dev))
        perm_r = torch.from_numpy(rng.permutation(n)).to(dev)
        inv = torch.empty_like(perm_r)
        inv[perm_r] = torch.arange(n, device=dev)
        r = torch.div(keys, n, rounding_mode="floor")
        keys = inv[r] * n + (keys - r * n)
        A = _csr_from_keys(keys, n, n, _values(rng, int(keys.numel()), prec), dev)
        n_rows = n_cols = n
    elif name == "4":
        nnz = _round_half_up(0.10 * n_rows * n_cols)
        keys = torch.from_numpy(rng.choice(n_rows * n_cols, size=nnz, replace=False)).to(dev)
        A = _csr_from_keys(keys, n_rows, n_cols, _values(rng, nnz, prec), dev)
    else:
        raise KeyError(name)
    bounds = np.append(np.arange(0, A.n_cols, cfg.delta, dtype=np.int64), A.n_cols)
    meta.update(nnz=A.nnz, n_rows=A.n_rows, n_cols=A.n_cols, scale=scale)
    return A, bounds, cfg, meta


def _blocked_host(rng, n: int, d: int, theta: float, prec: str):
    """Config 5's matrix (planted d x d blocks, rho = 1, no noise, rows scrambled) built straight in
    CSR order with numpy: identical arrays to ``make('5')`` (same draws in the same order) without
    sorting 687M keys.  Output row i is input row perm[i]; its columns are the 64 columns of every
    selected block of block row perm[i] // d, ascending."""
    bc = n // d
    n_sel = _round_half_up(theta * bc * bc)
    blocks = np.sort(rng.choice(bc * bc, size=n_sel, replace=False))
    perm_r = rng.permutation(n)
    b_row, b_col = blocks // bc, blocks % bc
    nblk = np.bincount(b_row, minlength=bc).astype(np.int64)
    start = np.zeros(bc + 1, np.int64)
    np.cumsum(nblk, out=start[1:])
    br = perm_r // d                       # input block row of every output row
    k = nblk[br]
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(k * d, out=row_ptr[1:])
    kp = np.zeros(n + 1, np.int64)
    np.cumsum(k, out=kp[1:])
    ent = np.repeat(start[br] - kp[:-1], k) + np.arange(int(kp[-1]), dtype=np.int64)
    col_idx = (b_col[ent][:, None] * d + np.arange(d, dtype=np.int64)[None, :]).reshape(-1)
    values = _values(rng, int(row_ptr[-1]), prec)
    return row_ptr, col_idx, values, n_sel * d * d


def make_host(name: str, scale: int = 1, precision: str | None = None):
    """Config ``name`` as host numpy CSR arrays -> (row_ptr, col_idx, values float64, boundaries, Config).

    Same matrix as ``make`` (bit-identical arrays); config 5 takes a sort-free numpy path, the others
    run ``make`` on the CPU.  Used by the CPU reference arm, which must not touch the GPU library."""
    cfg = CONFIGS[name]
    prec = precision or cfg.precision
    if name == "5":
        rng = np.random.default_rng(SEEDS[name])
        n = cfg.n_rows // scale
        row_ptr, col_idx, values, _ = _blocked_host(rng, n, 64, 0.01, prec)
        n_cols = n
    else:
        A, _, _, _ = make(name, scale=scale, device="cpu", precision=prec)
        row_ptr, col_idx, values = A.row_ptr.numpy(), A.col_idx.numpy(), A.values.numpy()
        n_cols = A.n_cols
    bounds = np.append(np.arange(0, n_cols, cfg.delta, dtype=np.int64), n_cols)
    return row_ptr, col_idx, values, bounds, cfg


def make_b(cfg: Config, n_cols: int, precision: str, device=None, seed: int = 1234) -> torch.Tensor:
    """B = U[0,1) rounded to the kernel dtype, [n_cols, N] row-major, on the device."""
    dev = _dev(device)
    g = torch.Generator(device="cpu").manual_seed(seed)
    B = torch.rand((n_cols, cfg.N), generator=g, dtype=torch.float32)
    dt = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}[precision]
    return B.to(dt).to(dev)

"""Benchmark: VBR SpMM effective GFLOP/s (2·nnz·N/s) on B200 vs the CPU reference path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

One "step" = one pass of the hot path's SpMM over the whole synthetic workload
(C = A·B with A resident as VBR tiles in HBM, B resident, C written in HBM).
Setup (synthesis, 1-SA, VBR build) runs before the timed region and is reported
under "stages".  For N>1 (torchrun) every rank owns a work-balanced shard of the
work list (whole block-row M-tiles: disjoint C rows, no data-path collective);
timing is the max over ranks.  See DESIGN.md §5 for the measurement protocol.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "VBR SpMM effective GFLOP/s (2·nnz·N/s) + tensor-pipe util, 1–8 B200 vs CPU ref"
L2_FLUSH_BYTES = 256 << 20


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="5")
    p.add_argument("--scale", type=int, default=1)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU time of the cpu_baseline sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=30)
    p.add_argument("--fused-gather", action="store_true",
                   help="N > 1: also time the fused all-gather (SpMM epilogues store into every rank's "
                        "symmetric-memory C over NVLink, dist.FusedGather) as 'gather_fused'")
    return p.parse_args()


# ---------------------------------------------------------------------------------------- helpers


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            if os.environ.get("RB_BENCH_SHARE_GPU"):  # functional test of the N > 1 path on one GPU
                local, backend = local % torch.cuda.device_count(), "gloo"
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


def _compact_h() -> int:
    from paper_2202_05868_b200 import config as rbconfig
    return rbconfig.compact_h()


def profile_traffic(config: str):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get(config)
    return None


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML every 5 ms while running."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------------------- CPU baseline


def reference_workload(name: str, scale: int, n_chunks: int):
    """The reference's CPU path on this config, built WITHOUT the GPU library: host CSR
    (synth.make_host: identical arrays to the GPU arm's), 1-SA by the C oracle (blocking.py:283-306),
    stored blocks and float64 payloads by the C oracle (vbr.py:88-125), B as float64.  The block rows
    are cut into ``n_chunks`` contiguous chunks of about equal VBR work; one timed step of the
    reference arm multiplies one chunk with the numpy restatement of spmm_vbr (multiply.py:72-97), so
    K steps over K chunks compute the whole product exactly once."""
    import oracle
    from paper_2202_05868_b200 import synth

    t0 = time.perf_counter()
    rp, ci, vals, bounds, cfg = synth.make_host(name, scale=scale)
    t1 = time.perf_counter()
    s = oracle.block_1sa_arrays(rp, ci, bounds, tau=cfg.tau, pruned=(name == "3"))
    perm, gp = s["row_perm"], s["group_ptr"]
    bp, bc = oracle.vbr_blocks(rp, ci, bounds, perm, gp)
    t2 = time.perf_counter()
    pay = oracle.vbr_payloads(rp, ci, vals, bounds, perm, gp, bp, bc)
    t3 = time.perf_counter()
    B = synth.make_b(cfg, len(bounds) and int(bounds[-1]), cfg.precision, device="cpu")
    B64 = B.float().numpy().astype(np.float64)
    n_rows, nnz, N = len(rp) - 1, int(rp[-1]), cfg.N
    # chunks of contiguous block rows, cut on the prefix sum of VBR-padded work (h * stored width)
    work = np.diff(np.asarray(gp, np.int64)) * group_widths(bounds, gp, bp, bc)
    cw = np.concatenate([[0], np.cumsum(work)])
    H = len(gp) - 1
    cuts = np.searchsorted(cw, np.linspace(0, cw[-1], n_chunks + 1), side="left")
    cuts[0], cuts[-1] = 0, H
    cuts = np.maximum.accumulate(cuts)
    row_nnz = np.diff(np.asarray(rp, np.int64))[np.asarray(perm, np.int64)]
    rn = np.concatenate([[0], np.cumsum(row_nnz)])
    gp64 = np.asarray(gp, np.int64)
    chunks = [(int(cuts[k]), int(cuts[k + 1]), int(rn[gp64[cuts[k + 1]]] - rn[gp64[cuts[k]]]))
              for k in range(n_chunks)]
    return dict(cfg=cfg, payloads=pay, row_perm=perm, row_partition=gp, bounds=bounds, B64=B64, n_rows=n_rows,
                n_cols=int(bounds[-1]), nnz=nnz, N=N, chunks=chunks, n_groups=H, n_blocks=len(bc),
                setup={"synth_host_s": round(t1 - t0, 2), "oracle_1sa_vbr_s": round(t2 - t1, 2),
                       "oracle_payloads_s": round(t3 - t2, 2)})


def time_chunk(w, k, threads, C):
    """One chunk of spmm_vbr (numpy restatement, multiply.py:72-97) -> seconds, useful flops."""
    import oracle

    from threadpoolctl import threadpool_limits

    lo, hi, nnz = w["chunks"][k]
    # one BLAS thread per worker thread: `threads` Python workers each calling a multi-threaded
    # OpenBLAS oversubscribe the cores (measured 7 vs 34 GFLOP/s on 8 cores, config 5 at 1/4 scale)
    with threadpool_limits(limits=1, user_api="blas"):
        t0 = time.perf_counter()
        oracle.spmm_vbr_np(w["payloads"], w["row_perm"], w["row_partition"], w["bounds"], w["B64"], threads=threads,
                           block_rows=range(lo, hi), out=C)
        return time.perf_counter() - t0, 2.0 * nnz * w["N"]


def group_widths(bounds, row_partition, blk_ptr, blk_col):
    w = np.diff(np.asarray(bounds, np.int64))
    bp = np.asarray(blk_ptr, np.int64)
    per_blk = w[np.asarray(blk_col, np.int64)] if len(blk_col) else np.zeros(0, np.int64)
    cs = np.concatenate([[0], np.cumsum(per_blk)])
    return cs[bp[1:]] - cs[bp[:-1]]


def host_info():
    """The CPU the baseline ran on (model, cpu_count, affinity, BLAS threads)."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            model = next((ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")), None)
    except OSError:
        pass
    try:
        affinity = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        affinity = None
    blas = {k: os.environ[k] for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS") if k in os.environ}
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity": affinity, "blas_env": blas,
            "blas_threads_per_worker": 1, "numpy": np.__version__}


def cpu_baseline(args, target_seconds, threads):
    """The reference CPU path (oracle structure + numpy spmm_vbr) on a bounded sample of the same
    workload: consecutive chunks (1/64 of the VBR work each) until ~target_seconds have been spent."""
    n_chunks = 64
    w = reference_workload(args.config, args.scale, n_chunks)
    C = np.zeros((w["n_rows"], w["N"]))
    spent, flops, done = 0.0, 0.0, 0
    while done < n_chunks and spent < target_seconds:
        t, f = time_chunk(w, done, threads, C)
        spent, flops, done = spent + t, flops + f, done + 1
    rows = w["chunks"][done - 1][1]
    return {"value": flops / spent / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "port",
            "seconds": round(spent, 3), "host": host_info(), "setup": w["setup"],
            "sample": f"reference path restated in oracle/ (C 1-SA + VBR build, numpy spmm_vbr of multiply.py:72-97, "
                      f"float64 per-block dgemm, threads={threads}): the first {done} of {n_chunks} equal-work chunks "
                      f"(block rows 0..{rows} of {w['n_groups']}) of the same matrix and B"}


# ---------------------------------------------------------------------------------------- main


def build_workload(args, device, world=1, rank=0):
    """Synthetic config on the device, 1-SA, VBR.  With world > 1 every rank runs the (deterministic)
    1-SA redundantly and builds only its own shard's VBR (dist.shard_vbr: the rows of its
    work-balanced range of block rows as a sub-matrix with its own tiles)."""
    from paper_2202_05868_b200 import dist as rbdist
    from paper_2202_05868_b200 import synth
    from paper_2202_05868_b200.device import DeviceVbr, block_1sa_device
    from paper_2202_05868_b200.types import MergePolicy

    t0 = time.perf_counter()
    dA, bounds, cfg, meta = synth.make(args.config, scale=args.scale, device=device)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pol = MergePolicy(tau=cfg.tau)
    dg = block_1sa_device(dA, bounds, pol, True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    shard = None
    if world == 1:
        dv = DeviceVbr.build(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=(cfg.precision,))
    else:
        dv, rows, ranges = rbdist.shard_vbr(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], cfg.precision,
                                            rank, world)
        shard = {"rows": rows, "ranges": ranges, "row_perm": dg.row_perm[: dA.n_rows].to(torch.int64)}
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    stages = {"synth_s": round(t1 - t0, 3), "block_1sa_s": round(t2 - t1, 4), "vbr_build_s": round(t3 - t2, 4),
              "n_groups": dg.n_groups, "n_blocks": dv.n_blocks}
    if shard:
        stages["shard_rows"] = list(shard["rows"])
    return dA, bounds, cfg, meta, dv, stages, shard


def run_ours(args, world, rank):
    from paper_2202_05868_b200 import _lib as L
    from paper_2202_05868_b200 import synth

    device = torch.device("cuda", torch.cuda.current_device())
    dA, bounds, cfg, meta, dv, stages, shard = build_workload(args, device, world, rank)
    prec = cfg.precision
    B = synth.make_b(cfg, dA.n_cols, prec, device=device)
    N = cfg.N
    C = torch.empty((dv.n_rows, N), dtype=torch.float32, device=device)  # this rank's rows (all at N=1)
    info = dv.plan_info(N, prec)
    launches_per_step = int(info["n_launches"])
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=device)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        dv.spmm(B, out=C, precision=prec)
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    sampler = ClockSampler(torch.cuda.current_device())
    barrier(world)
    torch.cuda.synchronize()
    with sampler:
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            starts[k].record(stream)
            dv.spmm(B, out=C, precision=prec)
            ends[k].record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms_local = sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / args.steps
    ms = allreduce_max(ms_local, world)
    useful = 2.0 * dA.nnz * N
    value = useful / (ms * 1e-3) / 1e9

    gather = run_gather(args, dv, B, C, prec, shard, world, flush, useful) if world > 1 else None
    gather_fused = run_gather_fused(args, dv, B, prec, shard, world, flush, useful) if (
        world > 1 and args.fused_gather) else None

    # ---- end to end through the reference-facing path: pinned float64 B -> device -> kernel -> float64 C
    e2e = run_e2e(args, dv, dA, B, prec, rank, world)
    csr = run_csr_comparator(args, dA, B, prec, flush) if world == 1 else None

    peaks = measured_peaks()
    useful_local = 2.0 * dv.csr.nnz * N  # this rank's kernel work (all of it at N=1)
    achieved_tflops = useful_local / (ms_local * 1e-3) / 1e12
    exec_tflops = info["executed_flops"] / (ms_local * 1e-3) / 1e12
    tensor_dominant = prec != "fp32" and info["core_vbr_flops"] < 0.5 * info["vbr_flops"]
    if tensor_dominant:
        roof = {"bound": "tensor", "kernel": ("spmm_tall2_kernel" if info["n_items_tall"] else
                                               "spmm_sweep_kernel" if info["n_sweep_steps"] else "spmm_short2_kernel"),
                "achieved": round(achieved_tflops, 3), "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                "frac": round(achieved_tflops / peaks["bf16_tflops"], 5), "traffic": profile_traffic(args.config),
                "peak_source": peaks["source"] + " (burst bf16, kernel timed alone)",
                "algorithmic": "2*nnz*N flops per launch",
                "executed_tflops": round(exec_tflops, 3),
                "executed_frac": round(exec_tflops / peaks["bf16_tflops"], 4),
                "executed_flops_per_launch": info["executed_flops"]}
    else:
        # CUDA-core (skinny / fp32) kernels gather B rows: HBM roofline on the minimal traffic of the
        # product — A read once (nnz x (value + 4 B column)), B read once, C written once (fp32).
        esz = 4 if prec == "fp32" else 2
        alg_bytes = dv.csr.nnz * (esz + 4) + dA.n_cols * N * esz + dv.n_rows * N * 4
        achieved_gbs = alg_bytes / (ms_local * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": ("spmm_simt_f32_kernel + skinny tiles" if prec == "fp32" else
                                            "spmm_csr_kernel over compact payloads" if _compact_h() else
                                            "spmm_skinny_staged_kernel (h<=4 classes)"),
                "achieved": round(achieved_gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved_gbs / peaks["hbm_gbs"], 5), "traffic": profile_traffic(args.config),
                "peak_source": peaks["source"] + " (HBM copy bandwidth)",
                "algorithmic": "nnz*(elem+4) + n_cols*N*elem + n_rows*N*4 bytes per step (all launches)",
                "algorithmic_bytes_per_step": alg_bytes,
                "executed_tflops": round(exec_tflops, 3),
                "useful_tflops": round(achieved_tflops, 4)}
        # The kernels these configs spend their time in gather one B row (N x elem bytes) per
        # nonzero, mostly from L2. That stream, not HBM, is what they saturate first. The
        # denominator is the random-row ld.global gather bandwidth that tools/l2bw/gather_probe
        # measured on B200 (profiles/r02/gather_probe.txt): 16.2-16.8 TB/s while B fits in L2,
        # 9.1-9.2 TB/s for a 256 MB B.
        gathered = dv.csr.nnz * N * esz
        b_bytes = dA.n_cols * N * esz
        peak_g = GATHER_L2_GBS if b_bytes <= 64 << 20 else GATHER_BIG_GBS
        roof["l2_gather"] = {"bytes_per_step": gathered,
                             "achieved_gbs": round(gathered / (ms_local * 1e-3) / 1e9, 1),
                             "peak_gbs": peak_g,
                             "frac": round(gathered / (ms_local * 1e-3) / 1e9 / peak_g, 4),
                             "what": "nnz x N x elem bytes of gathered B rows per step (one B row per "
                                     "nonzero) over the measured random-row gather bandwidth for B's size"}
    if roof["traffic"] and world == 1 and args.scale == 1:
        # the ncu DRAM bytes of one step over this run's step time: how close the step is to HBM
        roof["traffic_gbs"] = round(roof["traffic"] / (ms_local * 1e-3) / 1e9, 1)
        roof["traffic_frac_of_hbm"] = round(roof["traffic_gbs"] / peaks["hbm_gbs"], 4)
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": prec, "data": "synthetic",
        "config": workload_config(cfg, dA.n_rows, dA.n_cols, dA.nnz, world),
        "roofline": roof, "e2e": e2e, "gpu_launches": launches_per_step * args.steps, "gather": gather, "gather_fused": gather_fused,
        "csr_comparator": csr,
        "clocks": sampler.summary(),
        "stages": dict(stages, rho_prime=round(dA.nnz / max(dv.stored_area(), 1), 5),
                       padding_executed_over_useful=round(info["executed_flops"] / useful_local, 3),
                       padding_vbr_over_useful=round(info["vbr_flops"] / useful_local, 3)),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.config == "3" and args.scale == 1:  # the oracle's 1-SA alone takes minutes at 2^20
            out["cpu_baseline"] = {"skipped": "config 3's CPU structure (pruned C oracle 1-SA on R-MAT 2^20) takes "
                                              "~8 min per tau on one core; use --scale 16 for a CPU figure"}
        else:
            out["cpu_baseline"] = cpu_baseline(args, args.cpu_seconds, os.cpu_count() or 1)
    if rank == 0:
        print(json.dumps(out), flush=True)


# Random-row gather bandwidth (16 B per lane, 8 rows in flight per lane group, 4 CTAs/SM), measured
# by tools/l2bw/gather_probe on B200 (profiles/r02/gather_probe.txt): B in L2 (64 MB) / B of 256 MB
GATHER_L2_GBS, GATHER_BIG_GBS = 16500.0, 9150.0


def run_gather(args, dv, B, C, prec, shard, world, flush, useful):
    """N > 1: the optional collective of north_star / SURVEY §8(e) — NCCL all-gather of every rank's
    C rows plus the un-permute into source row order (dist.gather_c, multiply.py:90) — timed after
    the SpMM in the same step: SpMM + gather per step, max over ranks."""
    from paper_2202_05868_b200 import dist as rbdist

    steps = max(3, min(args.steps, 10))
    for _ in range(2):
        dv.spmm(B, out=C, precision=prec)
        full = rbdist.gather_c(C, shard["row_perm"], shard["ranges"])
    torch.cuda.synchronize()
    barrier(world)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s, e in ev:
        flush.zero_()
        s.record()
        dv.spmm(B, out=C, precision=prec)
        full = rbdist.gather_c(C, shard["row_perm"], shard["ranges"])
        e.record()
    torch.cuda.synchronize()
    ms = allreduce_max(sum(s.elapsed_time(e) for s, e in ev) / steps, world)
    del full
    return {"ms_per_step": round(ms, 4), "value": round(useful / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
            "what": "SpMM of the rank's shard + NCCL all-gather of C (fp32) + un-permute to source rows, "
                    "max over ranks; every rank ends with the full C"}


def run_gather_fused(args, dv, B, prec, shard, world, flush, useful):
    """N > 1, --fused-gather: the same product and collective result as run_gather, but the SpMM
    epilogues store each rank's rows at their source rows into every rank's symmetric-memory C over
    NVLink (rb_spmm_execute_fanout), then one device-side barrier: no NCCL call, no un-permute pass.
    Checked once against the NCCL path (bit-identical rows) before timing."""
    from paper_2202_05868_b200 import dist as rbdist

    try:
        fg = rbdist.FusedGather(int(shard["row_perm"].numel()), B.shape[1], B.device)
        C = torch.empty((dv.n_rows, B.shape[1]), dtype=torch.float32, device=B.device)
        dv.spmm(B, out=C, precision=prec)
        ref = rbdist.gather_c(C, shard["row_perm"], shard["ranges"])
        for _ in range(2):
            got = fg.run(dv, B, precision=prec)
        torch.cuda.synchronize()
        same = bool(torch.equal(got, ref))
        barrier(world)
        steps = max(3, min(args.steps, 10))
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for s, e in ev:
            flush.zero_()
            s.record()
            fg.run(dv, B, precision=prec)
            e.record()
        torch.cuda.synchronize()
        ms = allreduce_max(sum(s.elapsed_time(e) for s, e in ev) / steps, world)
        return {"ms_per_step": round(ms, 4), "value": round(useful / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                "matches_nccl_gather": same,
                "what": "SpMM of the rank's shard with fan-out epilogue stores into every rank's full C "
                        "(symmetric memory over NVLink) + device barrier, max over ranks"}
    except Exception as exc:  # noqa: BLE001 — report, do not lose the rest of the line
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


def run_csr_comparator(args, dA, B, prec, flush):
    """The paper's sparse baseline on the same device and inputs: spmm_csr (multiply.py:51-69) as
    the CSR gather kernel (csrc/csr.cu), same B, same L2 flush; not part of the headline value."""
    C = torch.empty((dA.n_rows, B.shape[1]), dtype=torch.float32, device=B.device)
    for _ in range(2):
        dA.spmm(B, out=C, precision=prec)
    steps = max(3, min(args.steps, 10))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s, e in ev:
        flush.zero_()
        s.record()
        dA.spmm(B, out=C, precision=prec)
        e.record()
    torch.cuda.synchronize()
    ms = sum(s.elapsed_time(e) for s, e in ev) / steps
    return {"kernel": "spmm_csr_kernel", "ms_per_step": round(ms, 5),
            "value": round(2.0 * dA.nnz * B.shape[1] / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s"}


def run_e2e(args, dv, dA, B, prec, rank, world):
    """Steps through the public host-buffer API (multiply.SpmmPipeline, what spmm_vbr_many runs):
    every step copies its float64 B from pinned host memory to the device, converts it, runs the
    SpMM, widens C to float64 and copies it back to pinned host memory (the reference's
    DenseMatrix contract, matrix.py:107-111).  Steps overlap on three streams (B of step k+1 in,
    SpMM of step k, C of step k-1 out); the timed region spans the first copy in to the last copy
    out, so every step's transfers are inside it."""
    from paper_2202_05868_b200.multiply import SpmmPipeline, pinned_dense

    N = B.shape[1]
    B_host = [B.double().cpu().pin_memory() for _ in range(2)]
    C_host = [pinned_dense(dv.n_rows, N) for _ in range(2)]
    pipe = SpmmPipeline(dv, N, prec)  # at N > 1: this rank's sub-VBR, so only its C rows come back
    for k in range(4):
        pipe.step(k, B_host[k % 2], C_host[k % 2])
    pipe.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(pipe.s_in)
    for k in range(args.e2e_steps):
        pipe.step(k, B_host[k % 2], C_host[k % 2])
    e.record(pipe.s_out)
    torch.cuda.synchronize()
    ms = allreduce_max(s.elapsed_time(e) / args.e2e_steps, world)
    return {"value": round(2.0 * dA.nnz * N / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s", "ms_per_step": round(ms, 4),
            "h2d_bytes_per_step": int(B_host[0].numel() * 8), "d2h_bytes_per_step": int(C_host[0].numel() * 8),
            "steps": args.e2e_steps,
            "path": "SpmmPipeline (spmm_vbr_many): pinned float64 B -> H2D -> rb_convert_f64 -> rb_spmm_execute "
                    "-> rb_widen_f32 -> D2H float64 C, steps overlapped on 3 streams"
                    + ("" if world == 1 else "; per rank: the whole B in, its shard's C rows out (no gather)")}


def run_reference(args, world, rank):
    """The reference's CPU implementation of the path on the host cores: oracle/ restatements only
    (C 1-SA and VBR build, numpy spmm_vbr), never librowblock_b200.so.  The K timed steps multiply K
    disjoint chunks of block rows (equal VBR work), so together they compute the whole product once."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_chunks = max(1, args.steps)
    w = reference_workload(args.config, args.scale, n_chunks)
    cfg = w["cfg"]
    C = np.zeros((w["n_rows"], w["N"]))
    for k in range(args.warmup):
        time_chunk(w, k % n_chunks, threads, C)
    C[:] = 0.0
    times, flops = [], 0.0
    for k in range(args.steps):
        t, f = time_chunk(w, k, threads, C)
        times.append(t)
        flops += f
    total = float(np.sum(times))
    ms = 1e3 * total / args.steps
    value = flops / total / 1e9
    desc = (f"reference path restated in oracle/ (C 1-SA + VBR build, numpy spmm_vbr of multiply.py:72-97, "
            f"float64 per-block dgemm, threads={threads}); the {args.steps} timed steps multiply {n_chunks} disjoint "
            f"equal-work chunks of block rows, i.e. the whole product once")
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(cfg, w["n_rows"], w["n_cols"], w["nnz"], world),
           "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": threads, "kind": "port",
                            "sample": desc, "host": host_info()},
           "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "stages": dict(w["setup"], n_groups=w["n_groups"], n_blocks=w["n_blocks"],
                          product_checksum=float(C.sum()))}
    print(json.dumps(out), flush=True)


def workload_config(cfg, n_rows, n_cols, nnz, world):
    """The `config` dict, identical in both arms."""
    return {"workload": f"config {cfg.name}: {cfg.description}", "n_rows": n_rows, "n_cols": n_cols, "nnz": nnz,
            "N": cfg.N, "delta": cfg.delta, "tau": cfg.tau, "policy": "jaccard, bounded, update",
            "parallelism": f"block-row shards x{world}" if world > 1 else "single GPU",
            "l2": "flushed between steps (256 MiB memset outside the timed events)"}


def main():
    args = parse()
    world, rank = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        if not torch.cuda.is_available():
            raise SystemExit("bench.py --impl ours needs a CUDA device")
        run_ours(args, world, rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()

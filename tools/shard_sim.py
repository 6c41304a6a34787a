"""Projected multi-GPU scaling on ONE GPU: time every shard's SpMM plan (rb_spmm_plan_create with
shard k of W, exactly what rank k runs under torchrun) back to back, take the max over shards.

    python tools/shard_sim.py <config> <W,W,...> [steps] [--plan]

Default: each shard is what bench.py --gpus W's rank k now runs — its own sub-VBR (dist.shard_vbr:
the rows of its work-balanced block-row range with their own tiles).  --plan times the older form,
shard k of W of one full plan (rb_spmm_plan_create(shard, n_shards)).

Prints, per W, the max / min shard time and the strong-scaling efficiency t1 / (W * max_k t_k)
of the sharded compute (B replicated, no collective; the optional C all-gather is separate)."""
import json, sys, torch
sys.path.insert(0, '.')
from paper_2202_05868_b200 import synth
from paper_2202_05868_b200.device import block_1sa_device, DeviceVbr
from paper_2202_05868_b200.types import MergePolicy

name = sys.argv[1]
worlds = [int(x) for x in sys.argv[2].split(',')]
steps = int(sys.argv[3]) if len(sys.argv) > 3 and not sys.argv[3].startswith("-") else 20
dA, bounds, cfg, meta = synth.make(name, scale=1, device="cuda")
dg = block_1sa_device(dA, bounds, MergePolicy(tau=cfg.tau), True)
dv = DeviceVbr.build(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], dtypes=(cfg.precision,))
B = synth.make_b(cfg, dA.n_cols, cfg.precision, device="cuda")
C = torch.empty((dA.n_rows, cfg.N), dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def time_shard(k, W):
    if W > 1 and "--plan" not in sys.argv:
        from paper_2202_05868_b200 import dist as rbdist
        sub, _, _ = rbdist.shard_vbr(dA, bounds, dg.row_perm, dg.group_ptr[: dg.n_groups + 1], cfg.precision, k, W)
        Cs = torch.empty((sub.n_rows, cfg.N), dtype=torch.float32, device="cuda")
        run = lambda: sub.spmm(B, out=Cs, precision=cfg.precision)  # noqa: E731
    else:
        run = lambda: dv.spmm(B, out=C, precision=cfg.precision, shard=k, n_shards=W)  # noqa: E731
    for _ in range(3):
        run()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s, e in ev:
        flush.zero_()
        s.record()
        run()
        e.record()
    torch.cuda.synchronize()
    return sum(s.elapsed_time(e) for s, e in ev) / steps


t1 = time_shard(0, 1)
out = {"config": name, "t1_ms": round(t1, 4), "worlds": {}}
for W in worlds:
    ts = [time_shard(k, W) for k in range(W)]
    out["worlds"][W] = {"max_ms": round(max(ts), 4), "min_ms": round(min(ts), 4),
                        "efficiency": round(t1 / (W * max(ts)), 4)}
    if "-v" in sys.argv:
        for k in range(W):
            info = dv.plan_info(cfg.N, cfg.precision, k, W)
            print(W, k, round(ts[k], 4), {f: info[f] for f in ("n_items_tall", "n_items_short", "n_items_skinny",
                                                                 "executed_flops", "row_begin_perm")}, flush=True)
print(json.dumps(out))

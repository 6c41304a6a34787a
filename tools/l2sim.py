"""Offline L2 model of the config-5 short-kernel schedules: replays the per-CTA access streams of a
schedule in (modelled) time order through an LRU cache and reports DRAM bytes for A tiles and B
panels.  Used to choose a schedule before spending GPU time; calibrated against the measured
17 GB/step of the round-1 schedule (ncu, profiles/r01_ncu_short2_cfg5.txt).

    python tools/l2sim.py --design current --slab 256 --l2mb 96
    python tools/l2sim.py --design sweep --slab 256 --slots 4 --l2mb 96
"""
import argparse
import heapq
from collections import OrderedDict

import numpy as np


def structure(nbr=4096, nbc=4096, dens=0.01, seed=5):
    rng = np.random.default_rng(seed)
    rows = []
    for g in range(nbr):
        k = rng.binomial(nbc, dens)
        rows.append(np.sort(rng.choice(nbc, size=k, replace=False)))
    return rows


def lpt(costs, ctas):
    order = np.argsort(-np.asarray(costs), kind="stable")
    heap = [(0.0, c) for c in range(ctas)]
    out = [[] for _ in range(ctas)]
    for i in order:
        t, c = heapq.heappop(heap)
        out[c].append(int(i))
        heapq.heappush(heap, (t + costs[i], c))
    return out


def streams_current(rows, slab, ctas, N=1024):
    """round-1: items (g, slab) slab-major, LPT onto CTAs; blocks ascending within an item."""
    per = [[] for _ in range(ctas)]
    for s in range(N // slab):
        a = lpt([len(r) for r in rows], ctas)
        for c in range(ctas):
            for g in a[c]:
                per[c].extend((g, t, int(b), s) for t, b in enumerate(rows[g]))
    return per


def streams_sweep(rows, slab, ctas, slots, N=1024, nbc=4096):
    """multi-slot merged circular sweep: each CTA holds `slots` rows; its blocks are processed in
    circular bcol order from a running phase; a finished slot takes the next row of the CTA's queue
    starting at the current phase (rotation)."""
    per = [[] for _ in range(ctas)]
    for s in range(N // slab):
        a = lpt([len(r) for r in rows], ctas)
        for c in range(ctas):
            queue = list(a[c])
            # interleave rows so that slot loads are spread: simple round-robin queue
            active = []  # [g, start_idx, consumed]
            phase = 0
            out = per[c]
            while queue or active:
                while len(active) < slots and queue:
                    g = queue.pop(0)
                    r = rows[g]
                    st = int(np.searchsorted(r, phase)) % max(len(r), 1)
                    active.append([g, st, 0])
                # pick the slot whose next bcol is closest ahead of the phase (circular)
                best, bd = None, None
                for k, (g, st, done) in enumerate(active):
                    r = rows[g]
                    b = int(r[(st + done) % len(r)])
                    d = (b - phase) % nbc
                    if bd is None or d < bd:
                        best, bd = k, d
                g, st, done = active[best]
                r = rows[g]
                t = (st + done) % len(r)
                b = int(r[t])
                out.append((g, t, b, s))
                phase = b
                active[best][2] += 1
                if active[best][2] == len(r):
                    active.pop(best)
    return per


def streams_snake(rows, slab, ctas, slots, N=1024, nbc=4096):
    """As streams_sweep, but the CTA's sweep reverses direction at the ends of the block-column
    range (boustrophedon): a row entering a slot collects its blocks ahead of the current column in
    the current direction, then the rest on the way back."""
    per = [[] for _ in range(ctas)]
    for s in range(N // slab):
        a = lpt([len(r) for r in rows], ctas)
        for c in range(ctas):
            queue = list(a[c])
            active = []  # [g, remaining set]
            phase, direction = 0, 1
            out = per[c]
            while queue or active:
                while len(active) < slots and queue:
                    g = queue.pop(0)
                    active.append([g, set(range(len(rows[g])))])
                best, bd = None, None
                for k, (g, rem) in enumerate(active):
                    r = rows[g]
                    for t in rem:
                        d = (r[t] - phase) * direction
                        if d >= 0 and (bd is None or d < bd):
                            best, bd = (k, t), d
                if best is None:  # nothing ahead: reverse
                    direction = -direction
                    continue
                k, t = best
                g, rem = active[k]
                b = int(rows[g][t])
                out.append((g, t, b, s))
                phase = b
                rem.discard(t)
                if not rem:
                    active.pop(k)
    return per


def replay(per, slab, l2mb, jitter=0.15, seed=0, a_bytes=8192, panel_rows=64, a_bypass=False):
    rng = np.random.default_rng(seed)
    b_bytes = panel_rows * slab * 2
    cap = l2mb << 20
    cache = OrderedDict()
    used = 0
    miss = {"A": 0, "B": 0}
    tot = {"A": 0, "B": 0}
    heap = [(rng.random(), c, 0) for c in range(len(per))]
    heapq.heapify(heap)
    while heap:
        t, c, i = heapq.heappop(heap)
        g, tt, b, s = per[c][i]
        for key, nb, kind in (((0, g, tt), a_bytes, "A"), ((1, b, s), b_bytes, "B")):
            tot[kind] += nb
            if kind == "A" and a_bypass:  # evict_first: streamed through, never displaces B
                miss[kind] += nb
                continue
            if key in cache:
                cache.move_to_end(key)
            else:
                miss[kind] += nb
                cache[key] = nb
                used += nb
                while used > cap:
                    _, v = cache.popitem(last=False)
                    used -= v
        if i + 1 < len(per[c]):
            heapq.heappush(heap, (t + 1.0 + jitter * rng.standard_normal(), c, i + 1))
    return {k: round(v / 1e9, 3) for k, v in miss.items()}, {k: round(v / 1e9, 3) for k, v in tot.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--design", default="current")
    ap.add_argument("--slab", type=int, default=256)
    ap.add_argument("--slots", type=int, default=4)
    ap.add_argument("--ctas", type=int, default=148)
    ap.add_argument("--l2mb", type=int, default=96)
    ap.add_argument("--jitter", type=float, default=0.15)
    ap.add_argument("--nbr", type=int, default=4096)
    ap.add_argument("--a-bypass", action="store_true")
    args = ap.parse_args()
    rows = structure(nbr=args.nbr)
    if args.design == "current":
        per = streams_current(rows, args.slab, args.ctas)
    elif args.design == "snake":
        per = streams_snake(rows, args.slab, args.ctas, args.slots)
    else:
        per = streams_sweep(rows, args.slab, args.ctas, args.slots)
    miss, tot = replay(per, args.slab, args.l2mb, args.jitter, a_bypass=args.a_bypass)
    print(vars(args), "DRAM miss GB", miss, "L2 GB", tot, "sum", round(sum(miss.values()), 2))


if __name__ == "__main__":
    main()

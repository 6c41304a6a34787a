"""Drop-in calls made inside a FORKED child of a process that already initialised CUDA.

The reference runs its sweep / curve points in process pools with the platform's default start
method (``fork`` on Linux: rb/metrics.py:122, rb/cli.py:199), and callers may do the same around the
drop-in.  CUDA cannot be used in such a child, so block_1sa / vbr_from_grouping / spmm_vbr forward the
call to one helper process per child, started with ``spawn``, which runs the same GPU code and
returns the (picklable, host-only) result.  The computation is still the device path: the helper
imports this package and calls the CUDA kernels through the C ABI; nothing runs on the CPU instead.
"""
from __future__ import annotations

import atexit
import multiprocessing as mp

_pool = None


def in_bad_fork() -> bool:
    import torch

    return bool(torch.cuda._is_in_bad_fork())


def _run(name, args, kwargs):
    import paper_2202_05868_b200 as rb

    return getattr(rb, name)(*args, **kwargs)


def call(name: str, *args, **kwargs):
    global _pool
    if _pool is None:
        _pool = mp.get_context("spawn").Pool(1)
        atexit.register(_pool.terminate)
    return _pool.apply(_run, (name, args, kwargs))

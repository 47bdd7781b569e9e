"""Multi-GPU sharding of one accumulate call.

One process per GPU.  The sample indices [first, first+count) are cut into
super-blocks of ``ABLMC_SUPERBLOCK`` samples; rank r computes a contiguous
range of super-blocks on its GPU (``ablmc_accumulate_partials``), ONE
collective (all-gather over ``torch.distributed``: NCCL on GPUs, gloo in the
CPU tests) moves the per-super-block partials, and every rank merges all of
them in index order (``ablmc_merge_partials``).  The merged bits are identical
for any world size, like the reference's worker-count invariance
(stats.hpp:93-95, test_estimators.cpp:97-108).
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np

from . import ablmc, capi


_collective_keepalive = None


def enable_collective(group=None) -> None:
    """Route every accumulate call of the library (and so every iteration of
    run_mlmc / run_stmc / decay_sweep) through this process group: each rank
    computes its contiguous super-block range and ONE all-gather per call
    (NCCL over NVLink for an "nccl" group; gloo on host for a CPU group)
    exchanges the partials (ablmc_set_collective in include/ablmc_b200.h)."""
    import torch
    import torch.distributed as dist

    global _collective_keepalive
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")

    def allgather(ctx, send, count, recv):
        try:
            src = np.ctypeslib.as_array(send, (count,))
            t = torch.from_numpy(src.copy()).to(dev)
            outs = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(outs, t, group=group)
            np.ctypeslib.as_array(recv, (world * count,))[:] = torch.cat(outs).cpu().numpy()
            return 0
        except Exception:  # noqa: BLE001 - reported to the C side as a failed collective
            return 1

    cb = capi.ALLGATHER_FN(allgather)
    _collective_keepalive = cb
    ablmc._check(ablmc.lib().ablmc_set_collective(rank, world, cb, None))


def disable_collective() -> None:
    global _collective_keepalive
    ablmc.lib().ablmc_set_collective(0, 1, capi.ALLGATHER_FN(), None)
    _collective_keepalive = None


def shard_superblocks(n_sb: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced super-block range [lo, hi) of `rank`."""
    base, extra = divmod(n_sb, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


PartialsFn = Callable[[ablmc.Problem, int, int, int, int, int], tuple]


def accumulate_sharded(acc: ablmc.LevelStats, first: int, count: int, pr: ablmc.Problem,
                       level: int, group=None, partials_fn: Optional[PartialsFn] = None,
                       superblock: int = capi.ABLMC_SUPERBLOCK) -> None:
    """accumulate_samples(acc, first, count, ., pr.level_sampler(level)) over
    all ranks of `group`; every rank ends with the same `acc`."""
    import torch
    import torch.distributed as dist

    if count <= 0:
        return
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n_sb = (count + superblock - 1) // superblock
    lo, hi = shard_superblocks(n_sb, rank, world)
    fn = partials_fn or (lambda p, l, f, c, a, b: ablmc.accumulate_partials(p, l, f, c, a, b))
    dim = pr.dim()
    if hi > lo:
        sums, cnts = fn(pr, level, first, count, lo, hi)
    else:
        sums, cnts = np.zeros((0, 2 * dim)), np.zeros((0, capi.ABLMC_NCOUNTS), dtype=np.int64)
    # pack (sums | counts as exact float64 bit patterns) into one buffer per rank
    width = 2 * dim + capi.ABLMC_NCOUNTS
    cap = (n_sb + world - 1) // world
    buf = np.zeros((cap, width))
    buf[: hi - lo, : 2 * dim] = sums
    buf[: hi - lo, 2 * dim:] = cnts.view(np.float64)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.from_numpy(buf).to(dev)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)  # the one collective
    allb = torch.stack(outs).cpu().numpy()
    rows = []
    for r in range(world):
        a, b = shard_superblocks(n_sb, r, world)
        rows.append(allb[r, : b - a])
    merged = np.concatenate(rows, axis=0)
    s = np.ascontiguousarray(merged[:, : 2 * dim])
    c = np.ascontiguousarray(merged[:, 2 * dim:]).view(np.int64)
    ablmc.merge_partials(acc, pr, level, s, c)

"""Multi-GPU sharding of accumulate calls.

The library shards natively (include/ablmc_b200.h, "multi-GPU sharding"):
sample indices are cut into super-blocks of ``ABLMC_SUPERBLOCK`` samples,
each rank computes a contiguous, balanced range of them, ONE all-gather per
accumulate call -- per ``accumulate_levels`` batch, i.e. per MLMC allocation
round -- moves the per-super-block partials, and every rank merges all of
them in index order.  The merged bits are identical for any world size, like
the reference's worker-count invariance (stats.hpp:120-135,
test_estimators.cpp:97-108).

This module only forms the group from Python:

* ``init_nccl_group`` -- one process per GPU (torchrun): rank 0's
  ``ncclUniqueId`` travels over the torch.distributed group, then the library
  joins its OWN NCCL communicator; the data path is device to device inside
  the library (no Python, no host staging);
* ``enable_collective`` -- a host all-gather callback over a torch.distributed
  group (gloo on CPU hosts, or ranks sharing a GPU);
* ``accumulate_sharded_levels`` -- the same exchange written out in Python
  around ``accumulate_partials`` (or any partials function: the CPU tests feed
  oracle partials), finishing with the library's own ``merge_gathered``.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

import numpy as np

from . import ablmc, capi


_collective_keepalive = None
collective_calls = 0  # host all-gathers issued through enable_collective's callback


def init_nccl_group(group=None, device: Optional[int] = None) -> None:
    """Join the library's native NCCL group: this process's GPU becomes rank
    ``dist.get_rank(group)`` of ``dist.get_world_size(group)``."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.cuda.current_device() if device is None else int(device)
    obj = [ablmc.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                               group=group)
    ablmc.init_group(dev, rank, world, obj[0])


def enable_collective(group=None) -> None:
    """Route every accumulate call of the library (and so every iteration of
    run_mlmc / run_stmc / decay_sweep) through this process group with a host
    all-gather callback (ablmc_set_collective): each rank computes its
    super-block range and ONE all-gather per call/batch exchanges the block
    of packed partials."""
    import torch
    import torch.distributed as dist

    global _collective_keepalive
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")

    def allgather(ctx, send, count, recv):
        global collective_calls
        collective_calls += 1
        try:
            src = np.ctypeslib.as_array(send, (count,))
            t = torch.from_numpy(src.copy()).to(dev)
            out = torch.empty(world * count, dtype=t.dtype, device=dev)
            dist.all_gather_into_tensor(out, t, group=group)
            np.ctypeslib.as_array(recv, (world * count,))[:] = out.cpu().numpy()
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


def accumulate_sharded_levels(requests: Sequence[tuple], pr: ablmc.Problem, group=None,
                              partials_fn: Optional[PartialsFn] = None,
                              superblock: int = capi.ABLMC_SUPERBLOCK,
                              fail_status: int = 0) -> None:
    """accumulate_levels over all ranks of `group` with ONE all-gather:
    requests are (acc, first, count, level); every rank ends with the same
    accs.  The block layout and the merge are the library's
    (gather_layout / merge_gathered); fail_status != 0 makes this rank
    report a failed share (every rank then raises)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    fn = partials_fn or (lambda p, l, f, c, a, b: ablmc.accumulate_partials(p, l, f, c, a, b))
    dim = pr.dim()
    n_sb = [max(0, (int(c) + superblock - 1) // superblock) for _, _, c, _ in requests]
    rows, width, base = ablmc.gather_layout(dim, world, n_sb)
    block = np.zeros(((rows + 1), width))
    status = fail_status
    if status == 0:
        try:
            for q, (acc, first, count, level) in enumerate(requests):
                lo, hi = shard_superblocks(n_sb[q], rank, world)
                if hi > lo:
                    sums, cnts = fn(pr, level, first, count, lo, hi)
                    block[base[q]: base[q] + hi - lo, : 2 * dim] = sums
                    block[base[q]: base[q] + hi - lo, 2 * dim:] = np.asarray(cnts, np.int64).view(
                        np.float64)
        except ablmc.CudaError:
            status = capi.ABLMC_ERR_CUDA
    block[rows, 0] = np.array([status], np.int64).view(np.float64)[0]
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.from_numpy(block.reshape(-1)).to(dev)
    out = torch.empty(world * t.numel(), dtype=t.dtype, device=dev)
    dist.all_gather_into_tensor(out, t, group=group)  # the one collective
    ablmc.merge_gathered([r[0] for r in requests], n_sb, world, out.cpu().numpy())


def accumulate_sharded(acc: ablmc.LevelStats, first: int, count: int, pr: ablmc.Problem,
                       level: int, group=None, partials_fn: Optional[PartialsFn] = None,
                       superblock: int = capi.ABLMC_SUPERBLOCK) -> None:
    """accumulate_samples(acc, first, count, ., pr.level_sampler(level)) over
    all ranks of `group`; every rank ends with the same `acc`."""
    accumulate_sharded_levels([(acc, first, count, level)], pr, group, partials_fn, superblock)

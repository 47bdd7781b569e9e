"""World-size-2 gloo tests (CPU) of the multi-GPU host path: super-block
sharding, the single all-gather, and the ordered merge through the product's
ablmc_merge_partials.  Per-super-block partials come from the C oracle here
(no GPU in this container); on the GPU box the same code takes them from
ablmc_accumulate_partials."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as O
from paper_1612_07717_b200 import ablmc
from paper_1612_07717_b200.sharding import (accumulate_sharded, accumulate_sharded_levels,
                                            shard_superblocks)

SB = 1000  # small super-blocks so a CPU-sized count spans several of them


def oracle_partials(pr, level, first, count, lo, hi):
    dim = pr.dim()
    sums = np.zeros((hi - lo, 2 * dim))
    cnts = np.zeros((hi - lo, 3), dtype=np.int64)
    for i, sb in enumerate(range(lo, hi)):
        a = sb * SB
        n = min(SB, count - a)
        st = O.Stats(dim)
        assert O.orc().orc_accumulate_samples(C.byref(pr._c), level, first + a, n, C.byref(st.c)) == 0
        sums[i, :dim], sums[i, dim:] = st.sum_y, st.sum_y2
        cnts[i] = (st.n, st.failed, st.cost_steps)
    return sums, cnts


def make_pr():
    q = ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=ablmc.equidistant_edges(4, 1.0))
    return ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.baoab, q, 0.05, 0.1, 1.0, 4, 3)


def worker(rank, world, port, count, out_q, mode="one"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pr = make_pr()
    if mode == "one":
        acc = ablmc.LevelStats().init(2, pr.h_level(2), pr.dim())
        accumulate_sharded(acc, 123, count, pr, 2, partials_fn=oracle_partials, superblock=SB)
        out_q.put((rank, acc.sum_y.tolist(), acc.sum_y2.tolist(), acc.n, acc.failed,
                   acc.cost_steps))
    elif mode == "batch":
        # one allocation round: three levels (one of them empty) in ONE all-gather
        reqs = [(ablmc.LevelStats().init(l, pr.h_level(l), pr.dim()), f, c, l)
                for l, f, c in ((0, 7, count), (1, 0, 0), (2, 123, count // 2 + 5))]
        accumulate_sharded_levels(reqs, pr, partials_fn=oracle_partials, superblock=SB)
        out_q.put((rank, [(a.sum_y.tolist(), a.sum_y2.tolist(), a.n, a.failed, a.cost_steps)
                          for a, *_ in reqs]))
    else:  # "fail": rank 1's share fails; every rank must get the error, none may hang
        acc = ablmc.LevelStats().init(2, pr.h_level(2), pr.dim())
        try:
            accumulate_sharded_levels([(acc, 123, count, 2)], pr, partials_fn=oracle_partials,
                                      superblock=SB, fail_status=4 if rank == 1 else 0)
            out_q.put((rank, "no error", acc.n))
        except ablmc.CudaError as e:
            out_q.put((rank, "error", str(e), acc.n))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_world(world, count, mode="one"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, count, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res)


def test_shard_ranges_cover_and_balance():
    for n_sb in (0, 1, 5, 8, 1000):
        for world in (1, 2, 3, 8):
            rs = [shard_superblocks(n_sb, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n_sb
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.timeout(300)
def test_two_ranks_match_one_rank_bit_for_bit():
    count = 4 * SB + 321  # 5 super-blocks, ragged tail, odd split across 2 ranks
    one = run_world(1, count)
    two = run_world(2, count)
    assert two[0][1:] == two[1][1:], "ranks disagree"
    assert two[0][1:] == one[0][1:], "world size changed the bits"
    # and equals the oracle's sums up to summation order
    pr = make_pr()
    st = O.Stats(pr.dim())
    assert O.orc().orc_accumulate_samples(C.byref(pr._c), 2, 123, count, C.byref(st.c)) == 0
    assert one[0][3] == st.n and one[0][5] == st.cost_steps
    assert np.allclose(one[0][1], st.sum_y, rtol=1e-12, atol=1e-12)


@pytest.mark.timeout(300)
def test_batch_of_levels_one_allgather_bit_for_bit():
    """Several levels (one empty) packed into ONE all-gather block (the
    library's gather_layout / merge_gathered): 2 and 3 ranks give the bits
    of 1 rank, level by level."""
    count = 3 * SB + 77
    one = run_world(1, count, "batch")
    for world in (2, 3):
        many = run_world(world, count, "batch")
        for r in many:
            assert r[1] == one[0][1], (world, r[0])
    (e0, e1, e2) = one[0][1]
    assert e1[2] == 0 and e1[4] == 0  # the empty request stays untouched
    pr = make_pr()
    for (lvl, first, c), got in zip(((0, 7, count), (2, 123, count // 2 + 5)), (e0, e2)):
        st = O.Stats(pr.dim())
        assert O.orc().orc_accumulate_samples(C.byref(pr._c), lvl, first, c, C.byref(st.c)) == 0
        assert got[2] == st.n and got[4] == st.cost_steps
        assert np.allclose(got[0], st.sum_y, rtol=1e-12, atol=1e-12)


@pytest.mark.timeout(300)
def test_failed_share_fails_every_rank_without_hanging():
    res = run_world(2, 2 * SB + 1, "fail")
    assert [r[1] for r in res] == ["error", "error"]
    assert all(r[3] == 0 for r in res)  # acc untouched on every rank
    assert "rank 1" in res[0][2]


def test_gather_layout_and_merge_host_only():
    """The block layout: cap_q = ceil(n_sb_q / world) rows per request, one
    status row; merge_gathered folds rank-major rows in global order."""
    rows, width, base = ablmc.gather_layout(2, 3, [5, 0, 1, 7])
    assert (rows, width, base) == (2 + 0 + 1 + 3, 2 * 2 + 3, [0, 2, 2, 3])
    # world 2, one request of 3 super-blocks: rank 0 owns 2, rank 1 owns 1
    dim, world = 1, 2
    rows, width, base = ablmc.gather_layout(dim, world, [3])
    assert rows == 2 and width == 5
    vals = [(1.0, 10.0, 4, 1, 40), (2.0, 20.0, 4, 0, 40), (0.5, 5.0, 2, 0, 20)]
    blocks = np.zeros((world, rows + 1, width))
    for sb, (s, s2, n, f, c) in enumerate(vals):
        w, r = (0, sb) if sb < 2 else (1, sb - 2)
        blocks[w, r, :2] = (s, s2)
        blocks[w, r, 2:] = np.array([n, f, c], np.int64).view(np.float64)
    acc = ablmc.LevelStats().init(1, 0.5, 1)
    ablmc.merge_gathered([acc], [3], world, blocks.reshape(-1))
    assert (acc.sum_y[0], acc.sum_y2[0], acc.n, acc.failed, acc.cost_steps) == (3.5, 35.0, 10, 1, 100)
    blocks[1, rows, 0] = np.array([3], np.int64).view(np.float64)[0]  # rank 1 reports a failure
    acc2 = ablmc.LevelStats().init(1, 0.5, 1)
    with pytest.raises(ablmc.SampleFailureError, match="rank 1"):
        ablmc.merge_gathered([acc2], [3], world, blocks.reshape(-1))
    assert acc2.n == 0

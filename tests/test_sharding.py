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
from paper_1612_07717_b200.sharding import accumulate_sharded, shard_superblocks

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


def worker(rank, world, port, count, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pr = make_pr()
    acc = ablmc.LevelStats().init(2, pr.h_level(2), pr.dim())
    accumulate_sharded(acc, 123, count, pr, 2, partials_fn=oracle_partials, superblock=SB)
    out_q.put((rank, acc.sum_y.tolist(), acc.sum_y2.tolist(), acc.n, acc.failed, acc.cost_steps))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_world(world, count):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, count, q)) for r in range(world)]
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

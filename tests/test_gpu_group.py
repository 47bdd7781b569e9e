"""The library's native multi-GPU path in ONE process (ablmc_init_devices:
one context and stream per GPU, an NCCL clique, one device-to-device
all-gather per accumulate call / per accumulate_levels batch): bit-identical
to the single-device calls.  On a one-GPU box the clique has one member, so
this exercises the packing, the NCCL all-gather, the status row and both
merges (host and device-resident) at world size 1; tests/test_sharding.py
covers the layout and merge for world sizes 2-3 on CPU, and the loopback
transport below (ablmc_init_loopback: n ranks sharing the one device, the
all-gather as device-to-device copies) runs the same workload at world sizes
2, 3 and 8 -- per-rank ranges, packed rows, status rows, both merges -- on the
device, everything but the NCCL call itself."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_1612_07717_b200 import ablmc

pytestmark = pytest.mark.gpu


def _device_result(pr, level, first, count):
    lib = ablmc.lib()
    ablmc._check(lib.ablmc_accumulate_device(C.byref(pr._c), level, first, count))
    d = ablmc.LevelStats().init(level, pr.h_level(level), pr.dim())
    v = d._view()
    ablmc._check(lib.ablmc_fetch_device_result(C.byref(pr._c), level, C.byref(v)))
    d._take(v)
    return d


def _key(s):
    return (s.sum_y.tobytes(), s.sum_y2.tobytes(), s.n, s.failed, s.cost_steps)


def _workload(pr, prb, count):
    out = {}
    a = ablmc.LevelStats().init(2, pr.h_level(2), 1)
    ablmc.accumulate_samples(a, 5, count, pr, 2)
    out["samples"] = _key(a)
    out["samples_collectives"] = ablmc.last_collective_count()
    reqs = [(ablmc.LevelStats().init(l, pr.h_level(l), 1), 7 * l, (count >> l) + l, l)
            for l in range(5)]
    ablmc.accumulate_levels(reqs, pr)
    out["levels"] = [_key(r[0]) for r in reqs]
    out["levels_collectives"] = ablmc.last_collective_count()
    b = ablmc.LevelStats().init(3, prb.h_level(3), prb.dim())
    ablmc.accumulate_samples(b, 11, count // 3, prb, 3)
    out["binned"] = _key(b)
    m = ablmc.run_mlmc(pr, 1e-3)
    out["mlmc"] = (m.estimate, m.stat_error, [_key(s) for s in m.level_stats])
    out["device"] = _key(_device_result(pr, 4, 3, count))
    out["empty"] = _key(_device_result(pr, 4, 3, 0))
    return out


def test_init_devices_native_nccl_is_bit_identical():
    n = torch.cuda.device_count()
    pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.gl, ablmc.QoISpec(), 0.05, 0.1,
                            1.0, 2, 21)
    q = ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=ablmc.equidistant_edges(16, 1.0))
    prb = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.baoab, q, 0.05, 0.1, 1.0, 4, 9)
    count = 3 * (1 << 22) + 777
    ablmc.init(0)
    single = _workload(pr, prb, count)
    assert single["samples_collectives"] == 0 and single["levels_collectives"] == 0
    try:
        ablmc.init_devices(n)
        info = ablmc.group_info()
        assert info == {"mode": 3, "rank": 0, "world": n, "n_local": n}
        grouped = _workload(pr, prb, count)
    finally:
        ablmc.init(0)
    # ONE all-gather per call, and per batch of five levels
    assert grouped["samples_collectives"] == 1 and grouped["levels_collectives"] == 1
    for k in single:
        if not k.endswith("collectives"):
            assert grouped[k] == single[k], k
    assert ablmc.group_info()["mode"] == 0


@pytest.mark.parametrize("world", [2, 3, 8])
def test_loopback_world_sizes_bit_identical(world):
    """World sizes > 1 on one GPU: the ranks' shares (some empty: requests of
    fewer super-blocks than ranks), the packed blocks, the device-resident
    grouped merge and the host merge give the single-device bits."""
    pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.gl, ablmc.QoISpec(), 0.05, 0.1,
                            1.0, 2, 21)
    q = ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=ablmc.equidistant_edges(16, 1.0))
    prb = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.baoab, q, 0.05, 0.1, 1.0, 4, 9)
    count = 5 * (1 << 22) + 777
    ablmc.init(0)
    single = _workload(pr, prb, count)
    try:
        ablmc.init_loopback(world, 0)
        assert ablmc.group_info() == {"mode": 3, "rank": 0, "world": world, "n_local": world}
        grouped = _workload(pr, prb, count)
    finally:
        ablmc.init(0)
    assert grouped["samples_collectives"] == 1 and grouped["levels_collectives"] == 1
    for k in single:
        if not k.endswith("collectives"):
            assert grouped[k] == single[k], k


def test_init_group_world_one_and_errors():
    ablmc.init(0)
    uid = ablmc.nccl_unique_id()
    assert len(uid) == 128 and any(uid)
    with pytest.raises(ValueError):
        ablmc.init_group(0, 1, 1, uid)  # rank out of range
    pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.se, ablmc.QoISpec(), 0.5, 0.1,
                            1.0, 1, 42)
    one = _device_result(pr, 10, 0, 1 << 22)
    try:
        ablmc.init_group(0, 0, 1, uid)
        assert ablmc.group_info()["mode"] == 2
        grp = _device_result(pr, 10, 0, 1 << 22)
        with pytest.raises(ValueError, match="native NCCL group"):
            from paper_1612_07717_b200 import capi
            ablmc._check(ablmc.lib().ablmc_set_collective(0, 1, capi.ALLGATHER_FN(lambda *a: 0), None))
    finally:
        ablmc.init(0)
    assert _key(grp) == _key(one)
    assert np.isfinite(one.mean())


def test_calls_from_several_host_threads_are_serialised():
    """Concurrent accumulate calls from four host threads (ctypes drops the
    GIL): the library's lock serialises them; every result equals the
    single-threaded one bit for bit."""
    import threading

    ablmc.init(0)
    prs = [ablmc.Problem.make(ablmc.ModelParams(), ig, ablmc.QoISpec(), 0.3 + 0.1 * i, 0.1, 1.0, 2,
                              100 + i)
           for i, ig in enumerate((ablmc.Integrator.se, ablmc.Integrator.gl, ablmc.Integrator.baoab,
                                   ablmc.Integrator.se))]
    jobs = [(i, level, 50000 + 1000 * level + i) for i in range(4) for level in (0, 1, 3, 5)]

    def run(i, level, count):
        a = ablmc.LevelStats().init(level, prs[i].h_level(level), 1)
        ablmc.accumulate_samples(a, 3 * i, count, prs[i], level)
        return _key(a)

    serial = {j: run(*j) for j in jobs}
    got, errs = {}, []

    def worker(i):
        try:
            for _ in range(5):
                for j in jobs:
                    if j[0] == i:
                        got[(j, _)] = run(*j)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    assert len(got) == 5 * len(jobs)
    for (j, _), k in got.items():
        assert k == serial[j], j

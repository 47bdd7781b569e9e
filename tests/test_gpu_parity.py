"""GPU parity: the sm_100a level sampler (through the C ABI) against the
reference's outputs (tests/golden/ref_vectors.json, bit-exact reference
fixtures) and the pinned C oracle.

Tolerances (north star: oracle mode within 1e-12 relative in fp64):
* host-supplied normals (oracle mode): SE bit-identical; GL/BAOAB within
  rel 1e-12 or abs 1e-13 (libdevice exp/expm1 vs glibc, <= 1-2 ulp);
  parity, reflection counts and ok flags exact.
* in-register Philox normals: the Philox words are integer-exact; Box-Muller
  log/sin/cos differ from glibc by ulps, so states within rel 1e-10 / abs 1e-12.
* per-level sums: rel 1e-11 (same samples, different but fixed summation
  tree); n, failed, cost_steps exact.
"""
import ctypes as C

import numpy as np
import pytest

import oracle_lib as O
from conftest import fx
from paper_1612_07717_b200 import ablmc, capi

pytestmark = pytest.mark.gpu

Ig = ablmc.Integrator


def make_problem(d, qoi=None):
    mp = ablmc.ModelParams(**{k: d[k] for k in ("kappa_sigma", "kappa_tau", "u_star", "H",
                                                  "eps_reg", "x_ref", "noise_scale")})
    if qoi is None:
        kind = ablmc.QoIKind(d.get("qoi_kind", 0))
        qoi = ablmc.QoISpec(kind=kind, bin_edges=d.get("edges", []))
    opt = ablmc.SampleOptions(signs_on=bool(d["signs_on"]), adaptive=bool(d.get("adaptive", 0)),
                              x_adapt=d.get("x_adapt", 0.05))
    return ablmc.Problem.make(mp, Ig(d["integrator"]), qoi, d["x0"], d["u0"], d["T"], d["m0"],
                              d["seed"], opt)


def close(a, b, rel, ab):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.all((np.abs(a - b) <= rel * np.abs(b)) | (np.abs(a - b) <= ab))


def stream_xi(seed, level, first, count, M):
    """The reference stream's normals (orc_normal_at is pinned bit-exact to
    NoiseStream::normal_at by tests/test_oracle.py)."""
    return np.array([O.orc_normals(seed, level, first + i, 0, M) for i in range(count)])


# ------------------------------------------------------------------ noise
def test_device_normals_vs_reference(ref_vectors):
    worst = 0.0
    for s in ref_vectors["normals"]:
        z = ablmc.normals(s["seed"], s["level"], s["idx"], s["k0"], len(s["z"]))
        want = np.array([fx(v) for v in s["z"]])
        assert close(z, want, 1e-13, 1e-15)
        worst = max(worst, float(np.max(np.abs(z - want) / np.abs(want))))
    print(f"max rel deviation of device Box-Muller normals: {worst:.3e}")


# ------------------------------------------------------------- oracle mode
@pytest.mark.parametrize("case_idx", range(16))
def test_pair_states_oracle_mode(ref_vectors, case_idx):
    case = ref_vectors["pairs"][case_idx]
    d = case["problem"]
    pr = make_problem(d)
    level, first = case["level"], case["first"]
    count = len(case["states"])
    M = d["m0"] << level
    xi = stream_xi(d["seed"], level, first, count, M)
    got = ablmc.simulate_pairs(pr, level, first, count, xi=xi)
    want = case["states"]
    ok = np.array([s[4] for s in want], bool)
    assert np.array_equal(got["fok"].astype(bool), ok), case["name"]
    g = got[ok]
    w = [s for s in want if s[4]]
    wx = np.array([[fx(s[0]), fx(s[1]), fx(s[5]), fx(s[6])] for s in w]).reshape(-1, 4)
    gx = np.stack([g["fx"], g["fu"], g["cx"], g["cu"]], axis=1)
    if d["integrator"] == 0:  # SE: no transcendental -> bit-identical
        assert np.array_equal(gx, wx), case["name"]
    else:
        assert close(gx, wx, 1e-12, 1e-13), (case["name"], np.max(np.abs(gx - wx)))
    assert [(s[2], s[3], s[7], s[8]) for s in w] == list(
        zip(g["fpar"].tolist(), g["fn"].tolist(), g["cpar"].tolist(), g["cn"].tolist()))


# uniform-grid cases; the adaptive golden cases (16-21) are the reference's
# ulp-sensitive schedule: pinned through the oracle (tests/test_oracle.py)
# and compared with the device in tests/test_gpu_adaptive.py
N_PAIRS = 16


@pytest.mark.parametrize("case_idx", range(N_PAIRS))
def test_pair_states_philox(ref_vectors, case_idx):
    case = ref_vectors["pairs"][case_idx]
    d = case["problem"]
    pr = make_problem(d)
    count = len(case["states"])
    got = ablmc.simulate_pairs(pr, case["level"], case["first"], count)
    want = case["states"]
    ok = np.array([s[4] for s in want], bool)
    assert np.array_equal(got["fok"].astype(bool), ok), case["name"]
    w = [s for s in want if s[4]]
    g = got[ok]
    wx = np.array([[fx(s[0]), fx(s[1]), fx(s[5]), fx(s[6])] for s in w]).reshape(-1, 4)
    gx = np.stack([g["fx"], g["fu"], g["cx"], g["cu"]], axis=1)
    assert close(gx, wx, 1e-10, 1e-12), (case["name"], np.max(np.abs(gx - wx)))
    assert [(s[2], s[3], s[7], s[8]) for s in w] == list(
        zip(g["fpar"].tolist(), g["fn"].tolist(), g["cpar"].tolist(), g["cn"].tolist()))


def test_survey_pair_kat():
    # simulate_pair(se, defaults, 0.5, 0.1, T=1, M=8, NoiseStream(42, 3, idx))
    pr = ablmc.Problem.make(ablmc.ModelParams(), Ig.se, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 42)
    s = ablmc.simulate_pairs(pr, 3, 0, 1)[0]
    assert close([s["fx"], s["fu"], s["cx"], s["cu"]],
                 [0.64579372369248766, 0.15921842792480534, 0.66134408294389468,
                  0.15499307057678519], 1e-12, 0)
    s = ablmc.simulate_pairs(pr, 3, 12345, 1)[0]
    assert close([s["fx"], s["fu"], s["cx"], s["cu"]],
                 [0.55708901811423728, 0.15391445097418696, 0.57230845534799446,
                  0.15126588419736006], 1e-12, 0)


@pytest.mark.parametrize("case_idx", [0, 1, 3, 4, 6, 7])  # uniform grid (2, 5, 8: adaptive)
def test_path_states(ref_vectors, case_idx):
    case = ref_vectors["paths"][case_idx]
    d = case["problem"]
    pr = make_problem(d)
    n = len(case["states"])
    want = np.array([[fx(s[0]), fx(s[1])] for s in case["states"]])
    assert not d.get("adaptive")
    for xi in (None, "stream"):
        x = None
        if xi:
            x = stream_xi(d["seed"], case["stream_level"], case["first"], n, case["M"])
        got = ablmc.simulate_paths(pr, case["M"], case["first"], n, case["stream_level"], xi=x)
        assert got["ok"].all()
        gx = np.stack([got["x"], got["u"]], axis=1)
        if xi and d["integrator"] == 0:
            assert np.array_equal(gx, want)
        else:
            assert close(gx, want, 1e-10 if xi is None else 1e-12, 1e-13)
        assert got["parity"].tolist() == [s[2] for s in case["states"]]
        assert got["n_refl"].tolist() == [s[3] for s in case["states"]]


def test_oracle_mode_arbitrary_xi_heavy_reflection():
    """Scaled normals drive many multi-wall reflections; GPU == C oracle."""
    rng = np.random.default_rng(3)
    mp = ablmc.ModelParams(u_star=1.0)
    for ig in (Ig.se, Ig.gl, Ig.baoab):
        pr = ablmc.Problem.make(mp, ig, ablmc.QoISpec(), 0.5, 0.0, 2.0, 16, 0)
        level, n = 5, 64
        M = 16 << level
        xi = rng.normal(size=(n, M)) * 2.0
        got = ablmc.simulate_pairs(pr, level, 0, n, xi=xi)
        p = O.default_params(u_star=1.0)
        for i in range(n):
            rc, f, c = O.orc_pair(int(ig), p, 0.5, 0.0, 2.0, M, 0, level, i, xi=xi[i])
            assert (rc == 0) == bool(got["fok"][i])
            if rc == 0:
                assert (got["fpar"][i], got["fn"][i], got["cpar"][i], got["cn"][i]) == (
                    f.parity, f.n_refl, c.parity, c.n_refl)
                v = [got["fx"][i], got["fu"][i], got["cx"][i], got["cu"][i]]
                if ig == Ig.se:
                    assert v == [f.x, f.u, c.x, c.u]
                else:
                    assert close(v, [f.x, f.u, c.x, c.u], 1e-12, 1e-13)
        assert got["fn"].sum() > 50


# -------------------------------------------------------- level sums
@pytest.mark.parametrize("case_idx", range(36))  # uniform grid (adaptive: test_gpu_adaptive)
def test_accumulate_vs_reference(ref_vectors, case_idx):
    case = ref_vectors["accumulate"][case_idx]
    d = case["problem"]
    pr = make_problem(d)
    dim = len(case["sum_y"])
    acc = ablmc.LevelStats().init(case["level"], pr.h_level(case["level"]), dim)
    ablmc.accumulate_samples(acc, case["first"], case["count"], pr, case["level"])
    assert (acc.n, acc.failed, acc.cost_steps) == (case["n"], case["failed"], case["cost_steps"])
    assert close(acc.sum_y, [fx(v) for v in case["sum_y"]], 1e-11, 1e-12)
    assert close(acc.sum_y2, [fx(v) for v in case["sum_y2"]], 1e-11, 1e-12)


def test_failures_counted_like_reference(ref_vectors):
    case = next(c for c in ref_vectors["pairs"] if c["name"] == "se_unstable_failures")
    d = case["problem"]
    pr = make_problem(d)
    n = len(case["states"])
    want_failed = sum(1 - s[4] for s in case["states"])
    acc = ablmc.LevelStats().init(1, pr.h_level(1), 1)
    ablmc.accumulate_samples(acc, 0, n, pr, 1)
    assert acc.failed == want_failed > 0
    assert acc.n == n - want_failed
    assert acc.cost_steps == acc.n * (4 + 2)  # failed samples contribute 0 steps
    with pytest.raises(ablmc.SampleFailureError):
        ablmc.check_failure_budget(acc)


def test_constant_qoi_difference_is_zero():
    # test_coupling.cpp:111-127
    q = ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=[0.0, 1.0])
    for ig in Ig:
        pr = ablmc.Problem.make(ablmc.ModelParams(), ig, q, 0.05, 0.1, 1.0, 40, 1)
        acc = ablmc.LevelStats().init(2, pr.h_level(2), 1)
        ablmc.accumulate_samples(acc, 7, 1, pr, 2)
        assert acc.n == 1 and acc.cost_steps == 160 + 80 and acc.sum_y[0] == 0.0
        acc = ablmc.LevelStats().init(2, pr.h_level(2), 1)
        ablmc.accumulate_samples(acc, 0, 5000, pr, 2)
        assert acc.sum_y[0] == 0.0 and acc.sum_y2[0] == 0.0


def test_binned_64_and_indicators_vs_oracle():
    edges = ablmc.equidistant_edges(64, 1.0)
    qs = [ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=edges),
          ablmc.QoISpec(kind=ablmc.QoIKind.smoothed_indicator),
          ablmc.QoISpec(kind=ablmc.QoIKind.raw_indicator)]
    for q in qs:
        for level in (0, 2):
            pr = ablmc.Problem.make(ablmc.ModelParams(), Ig.gl, q, 0.01, 0.1, 1.0, 10, 4)
            acc = ablmc.LevelStats().init(level, pr.h_level(level), q.size())
            ablmc.accumulate_samples(acc, 11, 6000, pr, level)
            ref = O.Stats(q.size())
            assert O.orc().orc_accumulate_samples(C.byref(pr._c), level, 11, 6000,
                                                  C.byref(ref.c)) == 0
            assert (acc.n, acc.failed, acc.cost_steps) == (ref.n, ref.failed, ref.cost_steps)
            assert close(acc.sum_y, ref.sum_y, 1e-11, 1e-11)
            assert close(acc.sum_y2, ref.sum_y2, 1e-11, 1e-11)


@pytest.mark.parametrize("bins,delta,uneven", [(256, 0.1, True), (37, 1e-12, True),
                                               (64, 0.3, False), (2, 0.05, False),
                                               (1024, 0.1, True), (1024, 0.002, False),
                                               (5000, 0.01, True)])
def test_binned_field_band_reduction_vs_oracle(bins, delta, uneven):
    """K4 (banded binned field): many bins, non-equidistant edges, a delta so
    small the band is disabled, a wide band, a 2-bin field, and fields wider
    than the old 256-bin cap (bin groups streamed through shared memory; 5000
    bins: edges read from global memory)."""
    rng = np.random.default_rng(bins)
    if uneven:
        inner = np.sort(rng.uniform(0.0, 1.0, bins - 1))
        edges = [0.0] + inner.tolist() + [1.0]
    else:
        edges = ablmc.equidistant_edges(bins, 1.0)
    q = ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=edges, delta=delta)
    for ig, level in ((Ig.gl, 0), (Ig.baoab, 3)):
        pr = ablmc.Problem.make(ablmc.ModelParams(), ig, q, 0.02, 0.1, 1.0, 4, 13)
        acc = ablmc.LevelStats().init(level, pr.h_level(level), bins)
        ablmc.accumulate_samples(acc, 5, 3000, pr, level)
        ref = O.Stats(bins)
        assert O.orc().orc_accumulate_samples(C.byref(pr._c), level, 5, 3000, C.byref(ref.c)) == 0
        assert (acc.n, acc.failed, acc.cost_steps) == (ref.n, ref.failed, ref.cost_steps)
        assert close(acc.sum_y, ref.sum_y, 1e-11, 1e-11)
        assert close(acc.sum_y2, ref.sum_y2, 1e-11, 1e-11)
        if level == 0:  # components of each sample sum to exactly 1 (qoi.hpp:153-156)
            assert abs(acc.sum_y.sum() - acc.n) <= 1e-9 * acc.n


# ---------------------------------------------- determinism / partitioning
def test_deterministic_and_add_merge():
    pr = ablmc.Problem.make(ablmc.ModelParams(), Ig.baoab, ablmc.QoISpec(), 0.05, 0.1, 1.0, 4, 9)
    a = ablmc.LevelStats().init(3, pr.h_level(3), 1)
    b = ablmc.LevelStats().init(3, pr.h_level(3), 1)
    ablmc.accumulate_samples(a, 0, 300_000, pr, 3)
    ablmc.accumulate_samples(b, 0, 300_000, pr, 3)
    assert a.sum_y[0] == b.sum_y[0] and a.sum_y2[0] == b.sum_y2[0] and a.n == b.n
    # continuing indices (first = attempts()) adds exactly the next samples
    c = ablmc.LevelStats().init(3, pr.h_level(3), 1)
    ablmc.accumulate_samples(c, 0, 100_000, pr, 3)
    ablmc.accumulate_samples(c, c.attempts(), 200_000, pr, 3)
    assert c.n == a.n and c.cost_steps == a.cost_steps
    assert abs(c.sum_y[0] - a.sum_y[0]) <= 1e-12 * abs(a.sum_y[0])


@pytest.mark.parametrize("level,m0", [(1, 2), (0, 1), (0, 4)])  # level 0, M <= 4: 4 samples/thread
def test_superblock_sharding_is_bit_identical(level, m0):
    pr = ablmc.Problem.make(ablmc.ModelParams(), Ig.gl, ablmc.QoISpec(), 0.05, 0.1, 1.0, m0, 21)
    count = 3 * capi.ABLMC_SUPERBLOCK + 12345  # ragged last super-block
    one = ablmc.LevelStats().init(level, pr.h_level(level), 1)
    ablmc.accumulate_samples(one, 17, count, pr, level)
    nsb = ablmc.num_superblocks(count)
    assert nsb == 4
    for split in ([0, 4], [0, 1, 4], [0, 2, 3, 4], [0, 1, 2, 3, 4]):
        parts = [ablmc.accumulate_partials(pr, level, 17, count, lo, hi)
                 for lo, hi in zip(split[:-1], split[1:])]
        sums = np.concatenate([p[0] for p in parts])
        cnts = np.concatenate([p[1] for p in parts])
        acc = ablmc.LevelStats().init(level, pr.h_level(level), 1)
        ablmc.merge_partials(acc, pr, level, sums, cnts)
        assert acc.sum_y[0] == one.sum_y[0] and acc.sum_y2[0] == one.sum_y2[0]
        assert (acc.n, acc.failed, acc.cost_steps) == (one.n, one.failed, one.cost_steps)


@pytest.mark.parametrize("ig", list(Ig))
@pytest.mark.parametrize("count,first", [(1, 0), (255, 3), (1023, 1), (1025, 4096 - 7), (70001, 11)])
def test_short_path_tiles_vs_oracle(ig, count, first):
    """Level 0 with M <= 4 runs 4 samples per thread (1024-sample tiles):
    ragged counts and offsets, every integrator, sums vs the oracle and counts
    exact (accumulate_samples, stats.hpp:96-136; level0_sample,
    coupling.hpp:228-244)."""
    for m0, u0 in ((1, 0.1), (3, 0.0), (4, 0.1)):
        pr = ablmc.Problem.make(ablmc.ModelParams(), ig, ablmc.QoISpec(), 0.05, u0, 1.0, m0, 5)
        acc = ablmc.LevelStats().init(0, pr.h_level(0), 1)
        ablmc.accumulate_samples(acc, first, count, pr, 0)
        ref = O.Stats(1)
        assert O.orc().orc_accumulate_samples(C.byref(pr._c), 0, first, count, C.byref(ref.c)) == 0
        assert (acc.n, acc.failed, acc.cost_steps) == (ref.n, ref.failed, ref.cost_steps)
        assert close(acc.sum_y, ref.sum_y, 1e-12, 1e-15)
        assert close(acc.sum_y2, ref.sum_y2, 1e-12, 1e-15)


@pytest.mark.parametrize("signs", [True, False])
@pytest.mark.parametrize("x0", [0.05, 0.5, 0.995])
def test_short_coupled_pairs_vs_oracle(signs, x0):
    """Coupled pairs of M = 2 fine steps (2 samples per thread, the one-window
    path only): near-ground and near-ceiling releases (SE failures, first-step
    reflections), coupling signs on/off, every integrator: counts exact
    (failed samples excluded, coupling.hpp:262-268), sums vs the oracle."""
    for ig in Ig:
        pr = ablmc.Problem.make(ablmc.ModelParams(), ig, ablmc.QoISpec(), x0, 0.1, 1.0, 1, 23,
                                ablmc.SampleOptions(signs_on=signs))
        acc = ablmc.LevelStats().init(1, pr.h_level(1), 1)
        ablmc.accumulate_samples(acc, 3, 20000, pr, 1)
        ref = O.Stats(1)
        assert O.orc().orc_accumulate_samples(C.byref(pr._c), 1, 3, 20000, C.byref(ref.c)) == 0
        assert (acc.n, acc.failed, acc.cost_steps) == (ref.n, ref.failed, ref.cost_steps), ig
        assert close(acc.sum_y, ref.sum_y, 1e-11, 1e-14)
        assert close(acc.sum_y2, ref.sum_y2, 1e-11, 1e-14)


@pytest.mark.parametrize("level,m0,first", [(0, 1, 2**32 - 1000), (2, 4, 2**32 - 1000),
                                            (1, 2, 2**40 + 17)])
def test_sample_indices_above_32_bits_vs_oracle(level, m0, first):
    """Index ranges crossing 2^32 and beyond 2^40 (the Philox counter's idx
    high word, noise.hpp:63-70): sums vs the oracle, device normals vs the
    oracle's stream."""
    for ig in Ig:
        pr = ablmc.Problem.make(ablmc.ModelParams(), ig, ablmc.QoISpec(), 0.05, 0.1, 1.0, m0, 9)
        acc = ablmc.LevelStats().init(level, pr.h_level(level), 1)
        ablmc.accumulate_samples(acc, first, 3000, pr, level)
        ref = O.Stats(1)
        assert O.orc().orc_accumulate_samples(C.byref(pr._c), level, first, 3000, C.byref(ref.c)) == 0
        assert (acc.n, acc.failed, acc.cost_steps) == (ref.n, ref.failed, ref.cost_steps)
        assert close(acc.sum_y, ref.sum_y, 1e-12, 1e-15)
        assert close(acc.sum_y2, ref.sum_y2, 1e-12, 1e-15)
    for idx in (2**32 - 1, 2**32, 2**40 + 3):
        z = ablmc.normals(9, level, idx, 0, 8)
        want = O.orc_normals(9, level, idx, 0, 8)
        assert np.all(np.abs(z - want) <= 1e-13 * np.abs(want) + 1e-15)


def test_device_resident_result_matches_host_path():
    pr = ablmc.Problem.make(ablmc.ModelParams(), Ig.se, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 42)
    lib = ablmc.lib()
    assert lib.ablmc_accumulate_device(C.byref(pr._c), 6, 0, 1_000_000) == 0
    dev = ablmc.LevelStats().init(6, pr.h_level(6), 1)
    v = dev._view()
    assert lib.ablmc_fetch_device_result(C.byref(pr._c), 6, C.byref(v)) == 0
    dev._take(v)
    host = ablmc.LevelStats().init(6, pr.h_level(6), 1)
    ablmc.accumulate_samples(host, 0, 1_000_000, pr, 6)
    assert dev.sum_y[0] == host.sum_y[0] and dev.n == host.n and dev.cost_steps == host.cost_steps


def test_edge_cases():
    pr = ablmc.Problem.make(ablmc.ModelParams(), Ig.gl, ablmc.QoISpec(), 0.05, 0.1, 1.0, 40, 5)
    acc = ablmc.LevelStats().init(1, pr.h_level(1), 1)
    ablmc.accumulate_samples(acc, 0, 1, pr, 1)
    assert acc.n == 1
    # huge first index (64-bit counter words) vs oracle
    for first in (2**40 + 1, 2**62):
        acc = ablmc.LevelStats().init(1, pr.h_level(1), 1)
        ablmc.accumulate_samples(acc, first, 4097, pr, 1)
        ref = O.Stats(1)
        assert O.orc().orc_accumulate_samples(C.byref(pr._c), 1, first, 4097, C.byref(ref.c)) == 0
        assert acc.n == ref.n and close(acc.sum_y, ref.sum_y, 1e-11, 1e-14)
    # odd path length (last Philox block half used) through accumulate_paths
    acc = ablmc.LevelStats().init(0, 1 / 7, 1)
    ablmc.accumulate_paths(acc, 3, 5000, pr, 7, 31)
    ref = O.Stats(1)
    assert O.orc().orc_accumulate_paths(C.byref(pr._c), 7, 31, 3, 5000, C.byref(ref.c)) == 0
    assert acc.n == ref.n and acc.cost_steps == ref.cost_steps
    assert close(acc.sum_y, ref.sum_y, 1e-11, 0)
    with pytest.raises(ValueError):
        ablmc.accumulate_samples(acc, 0, 10, pr, -1)
    # negative first: the reference feeds uint64(idx) to the stream (wraps)
    acc = ablmc.LevelStats().init(2, pr.h_level(2), 1)
    ablmc.accumulate_samples(acc, -3000, 5000, pr, 2)
    ref = O.Stats(1)
    assert O.orc().orc_accumulate_samples(C.byref(pr._c), 2, -3000, 5000, C.byref(ref.c)) == 0
    assert acc.n == ref.n and close(acc.sum_y, ref.sum_y, 1e-11, 1e-14)


def test_long_paths_level16_vs_oracle():
    """65536 fine + 32768 coarse steps per sample (M0 = 1, level 16)."""
    for ig in Ig:
        pr = ablmc.Problem.make(ablmc.ModelParams(), ig, ablmc.QoISpec(), 0.3, 0.1, 1.0, 1, 8)
        got = ablmc.simulate_pairs(pr, 16, 0, 24)
        p = O.default_params()
        for i in range(0, 24, 5):
            rc, f, c = O.orc_pair(int(ig), p, 0.3, 0.1, 1.0, 1 << 16, 8, 16, i)
            assert rc == 0 and got["fok"][i] == 1
            assert close([got["fx"][i], got["fu"][i], got["cx"][i], got["cu"][i]],
                         [f.x, f.u, c.x, c.u], 1e-9, 1e-11), (ig, i)
            assert (got["fn"][i], got["cn"][i]) == (f.n_refl, c.n_refl)


def test_multi_chunk_call_equals_superblock_merge():
    """A call spanning two launch chunks (chunk = 8 super-blocks for a scalar
    QoI) gives the same bits as merging independently computed super-blocks."""
    pr = ablmc.Problem.make(ablmc.ModelParams(), Ig.se, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 4)
    count = 9 * capi.ABLMC_SUPERBLOCK + 3
    one = ablmc.LevelStats().init(1, pr.h_level(1), 1)
    ablmc.accumulate_samples(one, 11, count, pr, 1)
    parts = [ablmc.accumulate_partials(pr, 1, 11, count, lo, hi) for lo, hi in ((0, 4), (4, 10))]
    acc = ablmc.LevelStats().init(1, pr.h_level(1), 1)
    ablmc.merge_partials(acc, pr, 1, np.concatenate([p[0] for p in parts]),
                         np.concatenate([p[1] for p in parts]))
    assert acc.sum_y[0] == one.sum_y[0] and acc.sum_y2[0] == one.sum_y2[0]
    assert (acc.n, acc.cost_steps) == (one.n, one.cost_steps) == (count, count * 3)


# ------------------------------------------------------- statistics
def test_level_statistics_vs_reference_same_streams():
    """Config-2 analogue: reference profile, x0 = 0.5, u0 = 0.1,
    M0 = 1, seed 42: GPU and reference see the same streams, so E[Y_l] and
    Var[Y_l] agree to rounding, far inside 3 combined standard errors."""
    R = O.ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    for ig in Ig:
        pr = ablmc.Problem.make(ablmc.ModelParams(), ig, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 42)
        for level in (1, 3, 6):
            n = 100_000
            g = ablmc.LevelStats().init(level, pr.h_level(level), 1)
            ablmc.accumulate_samples(g, 0, n, pr, level)
            r = O.Stats(1)
            assert R.ref_accumulate_samples(C.byref(pr._c), level, 0, n, 8, C.byref(r.c), None) == 0
            assert g.n == r.n and g.failed == r.failed
            assert abs(g.sum_y[0] - r.sum_y[0]) <= 1e-10 * abs(r.sum_y[0]) + 1e-12
            assert abs(g.sum_y2[0] - r.sum_y2[0]) <= 1e-10 * abs(r.sum_y2[0])


def test_mlmc_estimate_agrees_with_reference_independent_seeds():
    """run_mlmc on the device vs the reference's run_mlmc with a different
    seed: estimates within 3 combined standard errors + both bias bounds."""
    R = O.ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    eps = 1e-3
    pr = ablmc.Problem.make(ablmc.ModelParams(), Ig.gl, ablmc.QoISpec(), 0.05, 0.1, 1.0, 40, 555)
    g = ablmc.run_mlmc(pr, eps)
    pr2 = pr.with_seed(556)
    o = capi.MlmcOptionsC()
    ablmc.lib().ablmc_mlmc_options_defaults(C.byref(o))
    r = capi.RunResultC()
    assert R.ref_run_mlmc(C.byref(pr2._c), eps, C.byref(o), 16, C.byref(r)) == 0
    se = (g.stat_error[0] ** 2 + r.stat_error ** 2) ** 0.5
    assert abs(g.estimate[0] - r.estimate) <= 3 * se + g.bias_estimate + r.bias_estimate
    assert g.stat_error[0] ** 2 <= 0.5 * eps * eps * 1.0001  # completion contract
    assert g.failed_samples == 0 and g.levels_used >= 1


def test_cost_sweep_and_result_json_vs_reference():
    """cost_sweep (estimators.hpp:456-485) on the device against the
    reference's: same seeds -> same allocation -> identical cost_steps and
    estimates to rounding; the decay-sweep CSV is byte-identical when the
    statistics agree to all printed digits."""
    R = O.ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    pr = ablmc.Problem.make(ablmc.ModelParams(), Ig.gl, ablmc.QoISpec(), 0.05, 0.1, 1.0, 40, 99)
    eps = [1e-2, 4e-3]
    for method in ablmc.Method:
        got = ablmc.cost_sweep(pr, method, eps, (1.0, 0.5))
        rows = (capi.CostRowC * 2)()
        assert R.ref_cost_sweep(C.byref(pr._c), int(method), (C.c_double * 2)(*eps), 2, 1.0, 0.5,
                                8, rows) == 0
        for g, r in zip(got, rows):
            assert g.cost_steps == r.cost_steps
            assert abs(g.estimate - r.estimate) <= 1e-12 * abs(r.estimate)
    m = ablmc.run_mlmc(pr, 2e-3)
    js = ablmc.result_json(ablmc.RunConfig(timings=False, seed=99), m)
    assert '"schema_version": 1' in js and '"wall_seconds": 0.0' in js


def test_fast_div_sqrt_bit_identical_and_bm_libm_accuracy():
    """The branch-free fast div/sqrt equal __ddiv_rn/__dsqrt_rn bit for bit
    wherever they report no miss (2^26 random inputs incl. extreme
    exponents); the Box-Muller log/sincos kernels are within 1 ulp of
    libdevice (which is itself within 1-2 ulp of glibc)."""
    out = (C.c_uint64 * 15)()
    assert ablmc.lib().ablmc_selftest_fastmath(1 << 28, 12345, out) == 0
    (div_n, div_bad, div_miss, sq_n, sq_bad, sq_miss, log_ulp, sin_e, cos_e, exp_ulp, em1_ulp,
     em2_ulp, dc_n, dc_bad, bm1_bad) = list(out)
    assert dc_n == 1 << 28 and dc_bad == 0 and bm1_bad == 0
    print(f"div: {div_n} checked, {div_miss} misses; sqrt: {sq_n} checked, {sq_miss} misses; "
          f"log max ulp {log_ulp}; sin/cos max abs err {sin_e / 100}/{cos_e / 100} x 2^-53; "
          f"exp/expm1/expm1(2x) max ulp vs libdevice {exp_ulp}/{em1_ulp}/{em2_ulp}")
    assert div_n == sq_n == 1 << 28
    assert div_bad == 0 and sq_bad == 0
    assert 0 < div_miss < div_n // 4 + div_n // 8 and 0 < sq_miss < sq_n // 4
    assert log_ulp <= 2 and sin_e <= 200 and cos_e <= 200
    assert exp_ulp <= 2 and em1_ulp <= 2 and em2_ulp <= 3


def test_full_size_c5_properties():
    """BASELINE config 5 at the bench's full size (2^25 coupled paths, level 10,
    SE, reference profile): size-independent properties the oracle cannot
    check at this size -- exact counts and cost, bit-identical sums for one
    call vs an 8-way super-block split merged in order vs a rerun (the
    multi-GPU contract), and the coupled level's variance ratio to level 9
    near the strong-order-1/2 value 2^-1 ... 2^-2 band (Var[Y_l] ~ h^beta,
    beta in [1, 2])."""
    pr = ablmc.Problem.make(ablmc.ModelParams(), Ig.se, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 42)
    n = 1 << 25
    one = ablmc.LevelStats().init(10, pr.h_level(10), 1)
    ablmc.accumulate_samples(one, 0, n, pr, 10)
    assert (one.n, one.failed, one.cost_steps) == (n, 0, n * (1024 + 512))
    again = ablmc.LevelStats().init(10, pr.h_level(10), 1)
    ablmc.accumulate_samples(again, 0, n, pr, 10)
    assert (again.sum_y[0], again.sum_y2[0]) == (one.sum_y[0], one.sum_y2[0])
    nsb = ablmc.num_superblocks(n)
    assert nsb == 8
    parts = [ablmc.accumulate_partials(pr, 10, 0, n, k, k + 1) for k in range(nsb)]
    acc = ablmc.LevelStats().init(10, pr.h_level(10), 1)
    ablmc.merge_partials(acc, pr, 10, np.concatenate([p[0] for p in parts]),
                         np.concatenate([p[1] for p in parts]))
    assert (acc.sum_y[0], acc.sum_y2[0], acc.n, acc.cost_steps) == (
        one.sum_y[0], one.sum_y2[0], one.n, one.cost_steps)
    l9 = ablmc.LevelStats().init(9, pr.h_level(9), 1)
    ablmc.accumulate_samples(l9, 0, n // 4, pr, 9)
    ratio = one.variance() / l9.variance()
    assert 0.2 < ratio < 0.55, ratio
    assert abs(one.mean()) < 6 * one.std_error() + 1e-4  # E[Y_10] ~ c h: tiny


# ------------------------------------------ device elementary functions
# The only arithmetic not taken from the reference is the elementary
# functions (Box-Muller log/sin/cos, the OU exp/expm1), restated from fdlibm /
# Cody-Waite within 1-2 ulp of glibc.  With the oracle switched to the
# device's own restatement of them (orc_set_device_math) every integrator's
# path must be bit-identical: everything else is the reference's arithmetic.
def _params_of(d):
    return O.default_params(**{k: d[k] for k in ("kappa_sigma", "kappa_tau", "u_star", "H",
                                                   "eps_reg", "x_ref", "noise_scale")})


@pytest.fixture
def device_math():
    O.orc().orc_set_device_math(1)
    yield
    O.orc().orc_set_device_math(0)


@pytest.mark.parametrize("case_idx", range(16))
def test_pairs_bit_exact_given_device_math(ref_vectors, case_idx, device_math):
    case = ref_vectors["pairs"][case_idx]
    d = case["problem"]
    pr = make_problem(d)
    level, first = case["level"], case["first"]
    count = len(case["states"])
    M = d["m0"] << level
    p = _params_of(d)
    xi = stream_xi(d["seed"], level, first, count, M)  # glibc normals, host-supplied
    for mode, x in (("oracle", xi), ("philox", None)):
        got = ablmc.simulate_pairs(pr, level, first, count, xi=x)
        for i in range(count):
            rc, f, c = O.orc_pair(d["integrator"], p, d["x0"], d["u0"], d["T"], M, d["seed"],
                                  level, first + i, xi=None if x is None else x[i],
                                  signs_on=d["signs_on"])
            g = got[i]
            assert (rc == 0) == bool(g["fok"]), (case["name"], mode, i)
            if rc == 0:
                assert ([g["fx"], g["fu"], g["fpar"], g["fn"], g["cx"], g["cu"], g["cpar"], g["cn"]]
                        == [f.x, f.u, f.parity, f.n_refl, c.x, c.u, c.parity, c.n_refl]), (
                    case["name"], mode, i)


@pytest.mark.parametrize("ig", list(Ig))
def test_paths_and_sums_bit_exact_given_device_math(ig, device_math):
    pr = ablmc.Problem.make(ablmc.ModelParams(), ig, ablmc.QoISpec(kind=ablmc.QoIKind.smoothed_indicator),
                            0.05, 0.1, 1.0, 40, 77)
    got = ablmc.simulate_paths(pr, 40, 0, 256, 0)
    p = O.default_params()
    for i in range(256):
        rc, s = O.orc_path(int(ig), p, 0.05, 0.1, 1.0, 40, 77, 0, i)
        assert rc == 0 and [got["x"][i], got["u"][i], got["parity"][i], got["n_refl"][i]] == [
            s.x, s.u, s.parity, s.n_refl], i
    for level in (0, 3):
        acc = ablmc.LevelStats().init(level, pr.h_level(level), 1)
        ablmc.accumulate_samples(acc, 11, 9000, pr, level)
        st = O.Stats(1)
        assert O.orc().orc_accumulate_samples(C.byref(pr._c), level, 11, 9000, C.byref(st.c)) == 0
        assert (acc.n, acc.failed, acc.cost_steps) == (st.n, st.failed, st.cost_steps)
        # same samples bit for bit; only the summation tree differs
        assert close(acc.sum_y, st.sum_y, 1e-13, 1e-15)
        assert close(acc.sum_y2, st.sum_y2, 1e-13, 1e-15)


def test_accumulate_levels_batch_equals_sequential_calls():
    """ablmc_accumulate_levels (one device batch, one synchronisation; what
    the MLMC driver's allocation rounds use) == one accumulate_samples per
    level, bit for bit, incl. a multi-super-block level and a no-op."""
    pr = ablmc.Problem.make(ablmc.ModelParams(), Ig.baoab, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 3)
    reqs = [(0, 0, 70000), (3, 11, 5 * capi.ABLMC_SUPERBLOCK // 2), (1, 5, 0), (6, 0, 4097)]
    seq, bat = [], []
    for level, first, count in reqs:
        a = ablmc.LevelStats().init(level, pr.h_level(level), 1)
        a.sum_y[0], a.n = 1.25, 7  # add-merge into existing sums
        ablmc.accumulate_samples(a, first, count, pr, level)
        seq.append(a)
        b = ablmc.LevelStats().init(level, pr.h_level(level), 1)
        b.sum_y[0], b.n = 1.25, 7
        bat.append(b)
    ablmc.accumulate_levels([(b, f, c, l) for b, (l, f, c) in zip(bat, reqs)], pr)
    for a, b in zip(seq, bat):
        assert (a.sum_y.tolist(), a.sum_y2.tolist(), a.n, a.failed, a.cost_steps) == (
            b.sum_y.tolist(), b.sum_y2.tolist(), b.n, b.failed, b.cost_steps)


@pytest.mark.parametrize("x0,u0", [(0.5, float("nan")), (0.5, float("inf")), (1.5, 0.1),
                                   (11.0, 0.0), (0.0, -0.2), (1.0, 0.3), (-0.0, 0.2),
                                   (-0.0, -0.2), (-1e-300, 0.1)])
def test_degenerate_release_states_like_the_reference(x0, u0):
    """Release states the reference does not validate (model.hpp has no check
    on x0/u0): non-finite velocities fail every sample through reflect's
    finiteness test (particle.hpp:38-39), a release outside [0, H] is
    reflected on the first step or, beyond 10 H, fails; releases on the walls
    are inside.  Device == oracle (counts exact, sums within 1e-11)."""
    for ig in Ig:
        pr = ablmc.Problem.make(ablmc.ModelParams(), ig, ablmc.QoISpec(), x0, u0, 1.0, 40, 9)
        for level in (0, 2):
            acc = ablmc.LevelStats().init(level, pr.h_level(level), 1)
            ablmc.accumulate_samples(acc, 0, 3000, pr, level)
            st = O.Stats(1)
            assert O.orc().orc_accumulate_samples(C.byref(pr._c), level, 0, 3000,
                                                  C.byref(st.c)) == 0
            assert (acc.n, acc.failed, acc.cost_steps) == (st.n, st.failed, st.cost_steps), (
                ig, level)
            if st.n:
                assert close(acc.sum_y, st.sum_y, 1e-11, 1e-13)


@pytest.mark.parametrize("ig", list(Ig))
@pytest.mark.parametrize("prof", ["reference", "floored"])
def test_first_steps_hoisted_bit_exact_given_device_math(ig, prof):
    """Level 0 paths (M = 1..3) and level 1-3 pairs (M = 2..8) take their first
    step's sample-independent part from the host (KernelArgs::FirstStep,
    capi.cu first_step): device == oracle on the device's elementary
    functions, bit for bit, over releases inside, near and on the walls, with
    first half-steps that reflect (BAOAB), u0 = 0, signs on and off."""
    kw = {}
    if prof == "floored":
        kw = dict(profile=ablmc.Profile.floored, sigma_floor=1e-3, tau_min=1e-3, tau_max=1.0)
    O.orc().orc_set_device_math(1)
    try:
        for x0, u0, T in [(0.5, 0.1, 1.0), (0.02, -0.3, 1.0), (0.97, 0.4, 2.0), (0.0, -0.2, 1.0),
                          (1.0, 0.3, 1.0), (0.3, 0.0, 0.5), (0.01, -1.5, 1.0)]:
            for signs in (True, False):
                pr = ablmc.Problem.make(ablmc.ModelParams(), ig, ablmc.QoISpec(), x0, u0, T, 1, 5,
                                        ablmc.SampleOptions(signs_on=signs), **kw)
                c = pr._c
                O.orc().orc_set_profile(c.profile, c.const_sigma_u, c.const_tau, c.sigma_floor,
                                        c.tau_min, c.tau_max)
                for level in (1, 2, 3):
                    got = ablmc.simulate_pairs(pr, level, 1000, 64)
                    for i in range(64):
                        rc, f, cc = O.orc_pair(int(ig), c.params, x0, u0, T, 1 << level, 5, level,
                                               1000 + i, signs_on=int(signs))
                        assert (rc == 0) == bool(got["fok"][i]), (x0, u0, level, i)
                        if rc == 0:
                            assert [got["fx"][i], got["fu"][i], got["fpar"][i], got["fn"][i],
                                    got["cx"][i], got["cu"][i], got["cpar"][i], got["cn"][i]] == [
                                f.x, f.u, f.parity, f.n_refl, cc.x, cc.u, cc.parity, cc.n_refl], (
                                x0, u0, signs, level, i)
                for M in (1, 2, 3):
                    gp = ablmc.simulate_paths(pr, M, 77, 64, 0)
                    for i in range(64):
                        rc, s = O.orc_path(int(ig), c.params, x0, u0, T, M, 5, 0, 77 + i)
                        assert (rc == 0) == bool(gp["ok"][i]), (x0, u0, M, i)
                        if rc == 0:
                            assert [gp["x"][i], gp["u"][i], gp["parity"][i], gp["n_refl"][i]] == [
                                s.x, s.u, s.parity, s.n_refl], (x0, u0, M, i)
    finally:
        O.orc().orc_set_device_math(0)
        O.orc().orc_set_profile(0, 0, 0, 0, 0, 0)

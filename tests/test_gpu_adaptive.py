"""GPU parity of the adaptive (non-nested) sampler, SampleOptions::adaptive
(coupling.hpp:31-51 simulate_path_adaptive, 137-214 simulate_pair_adaptive),
against the C oracle, which tests/test_oracle.py pins bit-exact to the
reference (tests/golden/ref_vectors.json adaptive cases).

The reference's adaptive pair is itself sensitive to ulp-level changes of its
inputs: near the ground (tiny steps, many reflections) a 1-ulp change of the
normals can move a sample's end state by O(1) (measured on the oracle, which
is the reference bit for bit).  The device's in-register Box-Muller is within
ulps of glibc's, so per-sample parity is checked with the oracle driven by
the DEVICE's own normal stream (ablmc_normals: the kernel's Philox words and
Box-Muller), and
* SE: bit-identical states, parities, reflection counts, ok flags, steps and
  per-level sums (up to summation order) -- exact arithmetic end to end;
* GL/BAOAB: the OU weights use the device exp/expm1 (<= 1-2 ulp from glibc),
  so against the glibc oracle states agree within rel 1e-9 except on samples
  where the reference itself is ulp-sensitive: the fraction of differing
  samples may not exceed the reference's own sensitivity (oracle with device
  vs glibc normals) + 5% (+ 2 sigma of that count); with the oracle on the
  device's elementary functions too (orc_set_device_math) every integrator
  is bit-identical (test_adaptive_*_given_device_math).
Against the reference's own glibc-normal stream the level statistics agree
within their standard errors (test_adaptive_level_mean_vs_oracle).
"""
import ctypes as C

import numpy as np
import pytest

import oracle_lib as O
from paper_1612_07717_b200 import ablmc

pytestmark = pytest.mark.gpu
Ig = ablmc.Integrator


def close(a, b, rel, ab):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.all((np.abs(a - b) <= rel * np.abs(b)) | (np.abs(a - b) <= ab))


def problem(ig, x0=0.05, u0=0.1, T=1.0, m0=40, seed=5, x_adapt=0.05, signs_on=True, qoi=None,
            **mp):
    return ablmc.Problem.make(ablmc.ModelParams(**mp), ig, qoi or ablmc.QoISpec(), x0, u0, T, m0,
                              seed, ablmc.SampleOptions(signs_on=signs_on, adaptive=True,
                                                        x_adapt=x_adapt))


def dev_xi(seed, level, idx, K):
    """The device's NoiseStream(seed, level, idx) draws 0 .. K-1."""
    return ablmc.normals(seed, level, idx, 0, K)


def n_draws(steps, M):
    # a pair draws at most one normal per loop iteration and every iteration
    # ends with at least one step; a path draws one per step.  The margin
    # covers a different schedule under the device normals; max_iter bounds it.
    return min(2 * steps + 1024, 256 * M + 257)


def oracle_pair(c, level, idx, M):
    rc, f, cc, steps = O.orc_pair_adaptive(c.integrator, c.params, c.x0, c.u0, c.T, c.T / M,
                                           c.x_adapt, c.seed, level, idx, c.signs_on)
    xi = dev_xi(c.seed, level, idx, n_draws(steps if rc == 0 else 256 * M, M))
    rc, f, cc, steps = O.orc_pair_adaptive(c.integrator, c.params, c.x0, c.u0, c.T, c.T / M,
                                           c.x_adapt, c.seed, level, idx, c.signs_on, xi=xi)
    assert rc != 0 or steps < len(xi)  # enough draws supplied
    return rc, f, cc, steps


def oracle_path(c, stream_level, idx, M):
    rc, s, steps = O.orc_path_adaptive(c.integrator, c.params, c.x0, c.u0, c.T, c.T / M,
                                       c.x_adapt, c.seed, stream_level, idx)
    xi = dev_xi(c.seed, stream_level, idx, n_draws(steps if rc == 0 else 64 * M, M))
    rc, s, steps = O.orc_path_adaptive(c.integrator, c.params, c.x0, c.u0, c.T, c.T / M,
                                       c.x_adapt, c.seed, stream_level, idx, xi=xi)
    assert rc != 0 or steps <= len(xi)
    return rc, s, steps


CONFIGS = [
    dict(ig=Ig.se, x0=0.05, m0=40, x_adapt=0.05, level=2),
    dict(ig=Ig.gl, x0=0.05, m0=40, x_adapt=0.05, level=2),
    dict(ig=Ig.baoab, x0=0.05, m0=40, x_adapt=0.05, level=2),
    dict(ig=Ig.se, x0=0.012, m0=20, x_adapt=0.3, level=4),
    dict(ig=Ig.gl, x0=0.012, m0=20, x_adapt=0.3, level=4, signs_on=False),
    dict(ig=Ig.gl, x0=0.5, u0=0.0, T=2.0, m0=8, x_adapt=0.5, level=5, u_star=1.0),
    dict(ig=Ig.se, x0=0.5, u0=0.0, T=2.0, m0=16, x_adapt=0.5, level=5, u_star=1.0),
    dict(ig=Ig.baoab, x0=0.02, m0=10, x_adapt=0.5, level=3, eps_reg=0.005),
]


def differs(v, w):
    return not close(v, w, 1e-9, 1e-12)


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: f"{c['ig'].name}-l{c['level']}")
def test_adaptive_pairs_vs_oracle(cfg):
    cfg = dict(cfg)
    level = cfg.pop("level")
    pr = problem(seed=31, **cfg)
    c = pr._c
    n = 96
    got = ablmc.simulate_pairs(pr, level, 1000, n)
    M = c.m0 << level
    fails = flips = sensitive = 0
    for i in range(n):
        rc, f, cc, _ = oracle_pair(c, level, 1000 + i, M)
        g = got[i]
        v, w = [g["fx"], g["fu"], g["cx"], g["cu"]], [f.x, f.u, cc.x, cc.u]
        meta = (g["fpar"], g["fn"], g["cpar"], g["cn"]) == (f.parity, f.n_refl, cc.parity,
                                                            cc.n_refl)
        if c.integrator == 0:
            assert (rc == 0) == bool(g["fok"]), i
            assert rc != 0 or (meta and v == w), i
        else:
            rc2, f2, cc2, _ = O.orc_pair_adaptive(c.integrator, c.params, c.x0, c.u0, c.T, c.T / M,
                                                  c.x_adapt, c.seed, level, 1000 + i, c.signs_on)
            sensitive += (rc != rc2) or (rc == 0 and differs([f2.x, f2.u, cc2.x, cc2.u], w))
            flips += ((rc == 0) != bool(g["fok"])) or (rc == 0 and not (meta and not differs(v, w)))
        fails += rc != 0
    assert fails < n
    print(f"{cfg['ig'].name}: device/oracle differing samples {flips}/{n}, "
          f"reference ulp-sensitive samples {sensitive}/{n}")
    # both counts are one draw of an ulp-perturbation experiment: allow their
    # sampling noise (2 sigma) on top of 5%
    assert flips <= sensitive + 0.05 * n + 2 * np.sqrt(sensitive + 1)


@pytest.mark.parametrize("ig", [Ig.se, Ig.gl, Ig.baoab])
def test_adaptive_paths_vs_oracle(ig):
    pr = problem(ig, x0=0.015, m0=40, x_adapt=0.2, seed=8)
    c = pr._c
    n = 128
    got = ablmc.simulate_paths(pr, 40, 0, n, 0)
    flips = 0
    for i in range(n):
        rc, s, steps = oracle_path(c, 0, i, 40)
        assert rc == 0 and got["ok"][i]
        v, w = [got["x"][i], got["u"][i]], [s.x, s.u]
        meta = (got["parity"][i], got["n_refl"][i]) == (s.parity, s.n_refl)
        if ig == Ig.se:
            assert meta and v == w, i
        elif not (meta and close(v, w, 1e-9, 1e-12)):
            flips += 1
    assert flips <= 0.05 * n


def qoi_of(pr, x):
    c = pr._c
    poly = (C.c_double * 14)()
    O.orc().orc_build_smoothing_polynomial(c.qoi.r, poly)
    y = (C.c_double * 1)()
    O.orc().orc_evaluate(C.byref(c.qoi), poly, c.qoi.r, x, y)
    return y[0]


@pytest.mark.parametrize("ig", [Ig.se])
@pytest.mark.parametrize("level", [0, 3])
def test_adaptive_accumulate_vs_oracle(ig, level):
    """Per-level sums and the data-dependent cost (SampleOutcome::steps) of
    accumulate_samples against the oracle sample by sample (device normals)."""
    q = ablmc.QoISpec(kind=ablmc.QoIKind.smoothed_indicator)
    pr = problem(ig, x0=0.05, m0=20, x_adapt=0.1, seed=99, qoi=q)
    c = pr._c
    count, first = 1500, 17
    acc = ablmc.LevelStats().init(level, pr.h_level(level), 1)
    ablmc.accumulate_samples(acc, first, count, pr, level)
    M = c.m0 << level
    ys, cost, n = [], 0, 0
    for i in range(count):
        idx = first + i
        if level == 0:
            rc, s, steps = oracle_path(c, 0, idx, M)
            y = qoi_of(pr, s.x)
        else:
            rc, f, cc, steps = oracle_pair(c, level, idx, M)
            y = qoi_of(pr, f.x) - qoi_of(pr, cc.x)
        if rc == 0:
            ys.append(y)
            cost += steps
            n += 1
    ys = np.array(ys)
    assert acc.n == n and acc.failed == count - n
    uniform = count * M * (1.5 if level else 1.0)
    assert acc.cost_steps > uniform  # steps shrink near the ground
    assert acc.cost_steps == cost
    assert close(acc.sum_y, [ys.sum()], 1e-11, 1e-13)
    assert close(acc.sum_y2, [(ys * ys).sum()], 1e-11, 1e-13)


@pytest.mark.parametrize("ig", [Ig.se, Ig.gl, Ig.baoab])
def test_adaptive_level_mean_vs_oracle(ig):
    """Against the reference's own stream (glibc normals): level-2 mean and
    variance of Y agree within sampling error; mean steps within 0.5%."""
    q = ablmc.QoISpec(kind=ablmc.QoIKind.smoothed_indicator)
    pr = problem(ig, x0=0.05, m0=20, x_adapt=0.1, seed=7, qoi=q)
    count = 20000
    acc = ablmc.LevelStats().init(2, pr.h_level(2), 1)
    ablmc.accumulate_samples(acc, 0, count, pr, 2)
    st = O.Stats(1)
    assert O.orc().orc_accumulate_samples(C.byref(pr._c), 2, 0, count, C.byref(st.c)) == 0
    assert acc.failed == st.failed
    ma, mb = acc.sum_y[0] / acc.n, st.sum_y[0] / st.n
    va = acc.sum_y2[0] / acc.n - ma * ma
    assert abs(ma - mb) <= 3 * np.sqrt(2 * va / count) + 1e-15
    assert abs(acc.cost_steps - st.cost_steps) <= 5e-3 * st.cost_steps


def test_adaptive_binned_field_vs_oracle():
    q = ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=ablmc.equidistant_edges(16, 1.0))
    pr = problem(Ig.gl, x0=0.05, m0=20, x_adapt=0.1, seed=4, qoi=q)
    acc = ablmc.LevelStats().init(2, pr.h_level(2), 16)
    ablmc.accumulate_samples(acc, 0, 5000, pr, 2)
    st = O.Stats(16)
    assert O.orc().orc_accumulate_samples(C.byref(pr._c), 2, 0, 5000, C.byref(st.c)) == 0
    assert acc.n == st.n and abs(acc.cost_steps - st.cost_steps) <= 5e-3 * st.cost_steps
    # per-bin differences of the concentration field: within sampling error
    var = acc.sum_y2 / acc.n - (acc.sum_y / acc.n) ** 2
    assert np.all(np.abs(acc.sum_y / acc.n - st.sum_y / st.n) <= 4 * np.sqrt(2 * var / 5000) + 1e-12)


def test_adaptive_split_and_rerun_bit_identical():
    pr = problem(Ig.gl, x0=0.05, m0=40, seed=12)
    a = ablmc.LevelStats().init(3, pr.h_level(3), 1)
    ablmc.accumulate_samples(a, 0, 3 * 4096 + 77, pr, 3)
    b = ablmc.LevelStats().init(3, pr.h_level(3), 1)
    ablmc.accumulate_samples(b, 0, 3 * 4096 + 77, pr, 3)
    assert (a.sum_y.tolist(), a.sum_y2.tolist(), a.n, a.cost_steps) == (
        b.sum_y.tolist(), b.sum_y2.tolist(), b.n, b.cost_steps)


def test_adaptive_oracle_mode_rejected():
    pr = problem(Ig.se)
    with pytest.raises(ValueError, match="adaptive"):
        ablmc.simulate_pairs(pr, 1, 0, 4, xi=np.zeros((4, 80)))


def test_adaptive_mlmc_driver():
    """run_mlmc with adaptive levels: per-level cost is the measured step
    count, and the estimate agrees with the uniform-grid one (same limit)."""
    q = ablmc.QoISpec(kind=ablmc.QoIKind.smoothed_indicator)
    pa = problem(Ig.gl, x0=0.05, m0=20, x_adapt=0.1, seed=3, qoi=q)
    ra = ablmc.run_mlmc(pa, 2e-3)
    pu = ablmc.Problem.make(ablmc.ModelParams(), Ig.gl, q, 0.05, 0.1, 1.0, 20, 3)
    ru = ablmc.run_mlmc(pu, 2e-3)
    level_cost = sum(s.cost_steps for s in ra.level_stats)
    assert level_cost > 0 and ra.total_cost_steps >= level_cost
    assert abs(ra.estimate[0] - ru.estimate[0]) < 4 * (ra.stat_error[0] + ru.stat_error[0]) + 4e-3


def test_adaptive_golden_accumulate_statistics(ref_vectors):
    """The reference's own adaptive level sums (tests/golden/ref_vectors.json,
    glibc normals): counts exact, total steps within 0.1%, and every
    component's mean within 4 standard errors of the two runs' difference."""
    from test_gpu_parity import make_problem
    from conftest import fx
    cases = [c for c in ref_vectors["accumulate"] if c["problem"].get("adaptive")]
    assert len(cases) == 8
    for case in cases:
        pr = make_problem(case["problem"])
        dim = len(case["sum_y"])
        acc = ablmc.LevelStats().init(case["level"], pr.h_level(case["level"]), dim)
        ablmc.accumulate_samples(acc, case["first"], case["count"], pr, case["level"])
        assert (acc.n, acc.failed) == (case["n"], case["failed"])
        assert abs(acc.cost_steps - case["cost_steps"]) <= 1e-3 * case["cost_steps"]
        sy = np.array([fx(v) for v in case["sum_y"]])
        sy2 = np.array([fx(v) for v in case["sum_y2"]])
        n = acc.n
        var = np.maximum(sy2 / n - (sy / n) ** 2, 0.0)
        assert np.all(np.abs(acc.sum_y / n - sy / n) <= 4 * np.sqrt(2 * var / n) + 1e-12), case


@pytest.fixture
def device_math():
    O.orc().orc_set_device_math(1)
    yield
    O.orc().orc_set_device_math(0)


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: f"{c['ig'].name}-l{c['level']}")
def test_adaptive_pairs_bit_exact_given_device_math(cfg, device_math):
    """With the oracle on the device's own elementary functions
    (orc_set_device_math) and Philox stream, every integrator's adaptive pair
    is bit-identical: the GL/BAOAB pending increments are the reference's
    backward sums (pending terms kept per leg), so the only non-reference
    arithmetic left is log/sin/cos/exp/expm1."""
    cfg = dict(cfg)
    level = cfg.pop("level")
    pr = problem(seed=31, **cfg)
    c = pr._c
    n = 96
    got = ablmc.simulate_pairs(pr, level, 1000, n)
    M = c.m0 << level
    for i in range(n):
        rc, f, cc, _ = O.orc_pair_adaptive(c.integrator, c.params, c.x0, c.u0, c.T, c.T / M,
                                           c.x_adapt, c.seed, level, 1000 + i, c.signs_on)
        g = got[i]
        assert (rc == 0) == bool(g["fok"]), i
        if rc == 0:
            assert ([g["fx"], g["fu"], g["fpar"], g["fn"], g["cx"], g["cu"], g["cpar"], g["cn"]]
                    == [f.x, f.u, f.parity, f.n_refl, cc.x, cc.u, cc.parity, cc.n_refl]), i


@pytest.mark.parametrize("ig", [Ig.se, Ig.gl, Ig.baoab])
def test_adaptive_accumulate_given_device_math(ig, device_math):
    """Level sums of the persistent kernel (pending terms in shared memory,
    overflow recomputed by K1R) against the oracle on the device math: same
    samples, same steps; only the summation tree differs."""
    q = ablmc.QoISpec(kind=ablmc.QoIKind.smoothed_indicator)
    pr = problem(ig, x0=0.02, m0=20, x_adapt=0.3, seed=5, qoi=q)
    for level in (0, 3):
        acc = ablmc.LevelStats().init(level, pr.h_level(level), 1)
        ablmc.accumulate_samples(acc, 3, 4000, pr, level)
        st = O.Stats(1)
        assert O.orc().orc_accumulate_samples(C.byref(pr._c), level, 3, 4000, C.byref(st.c)) == 0
        assert (acc.n, acc.failed, acc.cost_steps) == (st.n, st.failed, st.cost_steps)
        assert close(acc.sum_y, st.sum_y, 1e-13, 1e-15)
        assert close(acc.sum_y2, st.sum_y2, 1e-13, 1e-15)

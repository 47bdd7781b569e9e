"""C-ABI checks that need no GPU: the library loads, exports every symbol the
public header declares, its struct layouts match the ctypes mirror, and the
host-side logic (validation, stability rule, failure budget, defaults)
behaves like the reference (model.hpp:37-47, qoi.hpp:119-141,
estimators.hpp:86-93, stats.hpp:139-143)."""
import ctypes as C
import re
import subprocess
import textwrap
from pathlib import Path

import numpy as np
import pytest

from paper_1612_07717_b200 import ablmc, capi

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "ablmc_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(ablmc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = capi.load()
    names = declared_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(capi.SIGNATURES), "ctypes mirror out of sync with the header"
    nm = subprocess.run(["nm", "-D", "--defined-only", str(capi.LIB_PATH)], capture_output=True,
                        text=True, check=True).stdout
    exported = set(re.findall(r" T (ablmc_\w+)", nm))
    assert set(names) <= exported


def test_abi_version():
    assert capi.load().ablmc_abi_version() == 2


def test_struct_layouts_match_header(tmp_path):
    structs = {"ablmc_problem": capi.ProblemC, "ablmc_level_stats": capi.LevelStatsC,
               "ablmc_pair_state": capi.PairStateC, "ablmc_run_result": capi.RunResultC,
               "ablmc_mlmc_options": capi.MlmcOptionsC, "ablmc_decay_row": capi.DecayRowC,
               "ablmc_qoi_spec": capi.QoISpecC}
    lines = [f'printf("{k} %zu\\n", sizeof({k}));' for k in structs]
    offs = {"ablmc_problem": ["qoi", "x0", "seed", "profile", "random_u0", "tau_max"],
            "ablmc_run_result": ["level_n", "level_sum_y2", "est_vec", "err_vec"]}
    for s, fields in offs.items():
        for f in fields:
            lines.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));')
    src = tmp_path / "l.c"
    src.write_text(textwrap.dedent(f"""
        #include <stdio.h>
        #include <stddef.h>
        #include "{HEADER}"
        int main(void) {{ {' '.join(lines)} return 0; }}"""))
    exe = tmp_path / "l"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    out = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                  check=True).stdout.splitlines())
    for k, cls in structs.items():
        assert int(out[k]) == C.sizeof(cls), k
    for s, fields in offs.items():
        cls = structs[s]
        for f in fields:
            assert int(out[f"{s}.{f}"]) == getattr(cls, f).offset, (s, f)


def test_problem_defaults_mirror_reference():
    pr = ablmc.Problem()
    c = pr._c
    assert (c.params.kappa_sigma, c.params.kappa_tau, c.params.u_star, c.params.H,
            c.params.eps_reg, c.params.x_ref, c.params.noise_scale) == (1.3, 0.5, 0.2, 1.0, 0.01,
                                                                         1.0, 1.0)
    assert (c.x0, c.u0, c.T, c.m0, c.seed, c.integrator) == (0.05, 0.1, 1.0, 40, 12345, capi.GL)
    assert (c.qoi.a, c.qoi.b, c.qoi.r, c.qoi.delta) == (0.1055, 0.1555, 4, 0.1)
    assert c.signs_on == 1 and c.adaptive == 0


def mk(**kw):
    mp = ablmc.ModelParams(**{k: kw.pop(k) for k in list(kw) if hasattr(ablmc.ModelParams, k)})
    qoi = kw.pop("qoi", ablmc.QoISpec())
    ig = kw.pop("ig", ablmc.Integrator.gl)
    return ablmc.Problem.make(mp, ig, qoi, kw.pop("x0", 0.05), 0.1, 1.0, kw.pop("m0", 40), 1,
                              **kw)


def test_validation_errors_mirror_reference():
    with pytest.raises(ValueError, match="eps_reg"):
        mk(eps_reg=0.6)  # test_model.cpp:51-54
    with pytest.raises(ValueError, match="positive"):
        mk(u_star=0.0)
    with pytest.raises(ValueError, match="x_ref"):
        mk(x_ref=2.0)
    with pytest.raises(ValueError, match="a < b"):
        mk(qoi=ablmc.QoISpec(kind=ablmc.QoIKind.raw_indicator, a=0.3, b=0.2))
    with pytest.raises(ValueError, match="span"):
        mk(qoi=ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=[0.1, 1.0]))
    with pytest.raises(ValueError, match="increasing"):
        mk(qoi=ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=[0.0, 0.5, 0.5, 1.0]))
    with pytest.raises(ValueError, match="r must be"):
        mk(qoi=ablmc.QoISpec(r=13))
    with pytest.raises(ValueError, match="adaptive"):
        mk(opt=ablmc.SampleOptions(adaptive=True), random_u0=True)
    with pytest.raises(ValueError, match="adaptive"):
        mk(opt=ablmc.SampleOptions(adaptive=True), fp32=True)
    with pytest.raises(ValueError, match="x_adapt"):
        mk(opt=ablmc.SampleOptions(adaptive=True, x_adapt=0.0))
    mk(opt=ablmc.SampleOptions(adaptive=True))  # coupling.hpp:137-214 on the device
    mk()  # defaults validate


def test_se_stability_rule():
    # estimators.hpp:86-93; test_estimators.cpp:158-162 (h = 0.05 >= 0.0387 is rejected)
    pr = mk(ig=ablmc.Integrator.se, m0=20)
    with pytest.raises(RuntimeError, match="symplectic Euler unstable"):
        pr.check_se_stability(0.05)
    pr.check_se_stability(0.025)
    mk(ig=ablmc.Integrator.gl).check_se_stability(1.0)  # only SE is checked


def test_failure_budget():
    st = ablmc.LevelStats().init(2, 0.1, 1)
    st.n, st.failed = 10000, 1
    ablmc.check_failure_budget(st)  # 1 <= 1e-4 * 10001
    st.failed = 2
    with pytest.raises(ablmc.SampleFailureError, match="level 2"):
        ablmc.check_failure_budget(st)


def test_h_level_and_dim():
    pr = mk(m0=40)
    assert pr.h_level(3) == 1.0 / 320
    q = ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=ablmc.equidistant_edges(64, 1.0))
    assert mk(qoi=q).dim() == 64


def test_level_stats_algebra():
    st = ablmc.LevelStats().init(0, 1.0, 1)  # test_estimators.cpp:305-315
    for v in (2.0, 4.0, 6.0):
        st.add([v], 1)
    assert st.mean() == 4.0 and st.variance() == 4.0
    assert abs(st.std_error() - (4.0 / 3.0) ** 0.5) <= 1e-14 * (4.0 / 3.0) ** 0.5


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    acc = ablmc.LevelStats().init(1, 0.0125, 1)
    with pytest.raises(ablmc.CudaError):
        ablmc.accumulate_samples(acc, 0, 100, mk(), 1)
    assert acc.n == 0


def test_count_zero_is_a_noop_without_touching_the_device():
    acc = ablmc.LevelStats().init(1, 0.0125, 1)
    ablmc.accumulate_samples(acc, 0, 0, mk(), 1)  # stats.hpp:99
    ablmc.accumulate_samples(acc, 0, -5, mk(), 1)
    assert acc.n == 0 and acc.sum_y[0] == 0.0


def test_merge_partials_is_ordered_add_merge():
    pr = mk()
    sums = np.array([[1.0, 1.0], [2.0, 4.0], [0.5, 0.25]])
    counts = np.array([[3, 0, 3 * 120], [4, 1, 4 * 120], [2, 0, 2 * 120]], dtype=np.int64)
    acc = ablmc.LevelStats().init(1, 0.0125, 1)
    acc.sum_y[0] = 10.0
    ablmc.merge_partials(acc, pr, 1, sums, counts)
    assert acc.sum_y[0] == ((10.0 + 1.0) + 2.0) + 0.5
    assert acc.sum_y2[0] == 1.0 + 4.0 + 0.25
    assert (acc.n, acc.failed, acc.cost_steps) == (9, 1, 9 * (80 + 40))


# ------------------------------------------- estimator helpers (host only)
def test_allocation_formula_goldens():
    # test_estimators.cpp:21-29
    assert ablmc.allocate_samples([1.0], [1.0], 0.1) == [200]
    assert ablmc.allocate_samples([1.0, 0.25], [1.0, 0.5], 0.1) == [342, 121]


def test_allocation_minimises_cost():
    # test_estimators.cpp:31-64: moving 20% of one level's samples and
    # restoring the error budget through another never costs less
    v, h, eps = [0.02, 6e-4, 1.5e-4], [0.025, 0.0125, 0.00625], 1e-3
    budget = 0.5 * eps * eps
    s = sum((v[l] / h[l]) ** 0.5 for l in range(3))
    n = [2.0 / (eps * eps) * (v[l] * h[l]) ** 0.5 * s for l in range(3)]
    assert ablmc.allocate_samples(v, h, eps) == [int(np.ceil(x)) for x in n]

    def cost(m):
        return sum(m[l] / h[l] for l in range(3))

    def err2(m):
        return sum(v[l] / m[l] for l in range(3))

    assert abs(err2(n) / budget - 1.0) <= 1e-12
    for down in range(3):
        for up in range(3):
            if up == down:
                continue
            m = list(n)
            m[down] *= 0.8
            rest = err2(m) - v[up] / m[up]
            if rest >= budget:
                continue
            m[up] = v[up] / (budget - rest)
            assert cost(m) >= cost(n) * (1.0 - 1e-12)


def test_bias_constant_fit_on_exact_power_laws():
    # test_estimators.cpp:66-88
    hs = [0.025, 0.0125, 0.00625, 0.003125]
    f = ablmc.estimate_bias_constants(hs, [0.5 * h for h in hs], [1e-9] * 4)
    assert abs(f.alpha - 1.0) <= 1e-10 and abs(f.c1 - 0.5) <= 1e-10
    f = ablmc.estimate_bias_constants(hs, [3.0 * h * h for h in hs], [1e-12] * 4)
    assert abs(f.alpha - 2.0) <= 1e-10 and abs(f.c1 - 1.0) <= 1e-10
    with pytest.raises(RuntimeError, match="indistinguishable"):
        ablmc.estimate_bias_constants([0.01] * 3, [1e-6] * 3, [1e-6] * 3)
    with pytest.raises(ValueError, match="at least 3"):
        ablmc.estimate_bias_constants(hs[:2], [1.0, 2.0], [0.0, 0.0])


def test_level_selection():
    # test_estimators.cpp:90-97
    assert ablmc.choose_levels(1.0, 1.0, 0.01, 40, 1.0) == 2
    assert ablmc.choose_levels(1.0, 1.0, 10.0, 40, 1.0) == 0
    for eps in (0.01, 0.003, 0.001):
        assert ablmc.choose_levels(2.0, 1.0, eps, 40, 1.0) <= ablmc.choose_levels(1.0, 1.0, eps,
                                                                                  40, 1.0)
    with pytest.raises(RuntimeError):
        ablmc.choose_levels(1.0, 1.0, 1e-9, 40, 1.0, 4)
    with pytest.raises(ValueError):
        ablmc.choose_levels(0.0, 1.0, 0.01, 40, 1.0)


def test_fit_power_law():
    e, lp = ablmc.fit_power_law([0.1, 0.05, 0.025], [3 * 0.1 ** 1.5, 3 * 0.05 ** 1.5,
                                                      3 * 0.025 ** 1.5])
    assert abs(e - 1.5) <= 1e-12 and abs(np.exp(lp) - 3.0) <= 1e-12
    with pytest.raises(ValueError, match="positive"):
        ablmc.fit_power_law([0.1, 0.05], [1.0, 0.0])
    with pytest.raises(ValueError, match="two points"):
        ablmc.fit_power_law([0.1], [1.0])


def test_adaptive_step_size_goldens():
    # test_coupling.cpp:18-25
    mp = ablmc.ModelParams()
    assert ablmc.adaptive_step_size(0.5, 0.025, 0.05, mp) == 0.025
    assert ablmc.adaptive_step_size(0.05, 0.025, 0.05, mp) == 0.025
    v = ablmc.adaptive_step_size(0.01, 0.025, 0.05, mp)
    assert abs(v - 0.19390825748466839 * 0.025) <= 1e-12 * 0.19390825748466839 * 0.025


def test_smoothing_polynomial_product_vs_goldens_and_criterion_9():
    """The product's host polynomial (used by the device QoI): the
    reference's golden coefficients (test_qoi.cpp:33-59) bit for bit vs the
    pinned oracle, and acceptance criterion 9 (acceptance.cpp:367-391): r = 2
    coefficients (1/2, -9/8, 0, 5/8) to 1e-12, g(-1) = 1, g(1) = 0 and the
    moment conditions to 1e-10 for r <= 8."""
    import oracle_lib as O
    for r in range(0, 13):
        got = ablmc.build_smoothing_polynomial(r)
        c = (C.c_double * (r + 2))()
        assert O.orc().orc_build_smoothing_polynomial(r, c) == 0
        assert got == list(c), r
    p2 = ablmc.build_smoothing_polynomial(2)
    assert max(abs(a - b) for a, b in zip(p2, [0.5, -1.125, 0.0, 0.625])) <= 1e-12
    worst = 0.0
    for r in range(0, 9):
        p = ablmc.build_smoothing_polynomial(r)
        ev = lambda s: sum(ci * s ** i for i, ci in enumerate(p))  # noqa: E731
        worst = max(worst, abs(ev(-1.0) - 1.0), abs(ev(1.0)))
        for j in range(r):
            m = sum(p[i] * 2.0 / (i + j + 1) for i in range(len(p)) if (i + j) % 2 == 0)
            worst = max(worst, abs(m - (1.0 if j % 2 == 0 else -1.0) / (j + 1)))
    assert worst <= 1e-10
    with pytest.raises(ValueError, match="r must be"):
        ablmc.build_smoothing_polynomial(13)


def test_release_coeffs_equal_the_oracle_bit_for_bit():
    """The samplers take every path's first-step sde_coeffs(x0) from the host
    (capi.cu host_coeffs); they must be the reference's IEEE values bit for
    bit (model.hpp:73-89; extension profiles as restated by the oracle), for
    release heights inside, on the clamp boundaries, on the walls and outside
    the layer, and for non-power-of-two H."""
    import oracle_lib as O
    lib = capi.load()
    rng = np.random.default_rng(7)
    out = (C.c_double * 4)()
    cases = 0
    for trial in range(400):
        H = float(rng.choice([1.0, 2.0, 3.0, 0.75]))
        mp = ablmc.ModelParams(kappa_sigma=float(rng.uniform(0.8, 2.0)),
                               kappa_tau=float(rng.uniform(0.3, 0.9)),
                               u_star=float(rng.choice([0.1, 0.2, 1e-12])), H=H,
                               eps_reg=float(rng.choice([0.005, 0.01, 0.05])) * H, x_ref=H,
                               noise_scale=float(rng.choice([1.0, 0.5])))
        prof = ablmc.Profile(int(rng.integers(0, 3)))
        kw = dict(const_sigma_u=1.3, const_tau=float(rng.choice([0.1, 0.5])), sigma_floor=1e-3,
                  tau_min=1e-3, tau_max=1.0) if prof != ablmc.Profile.reference else {}
        x0 = float(rng.choice([rng.uniform(0, 1), 0.0, 1.0, mp.eps_reg / H, 1 - mp.eps_reg / H,
                               1.5, -0.01])) * H
        pr = ablmc.Problem.make(mp, ablmc.Integrator.gl, ablmc.QoISpec(), x0, 0.1, 1.0, 4, 1,
                                profile=prof, **kw)
        assert lib.ablmc_release_coeffs(C.byref(pr._c), out) == 0
        c = pr._c
        O.orc().orc_set_profile(c.profile, c.const_sigma_u, c.const_tau, c.sigma_floor,
                                c.tau_min, c.tau_max)
        try:
            ref = O.orc().orc_sde_coeffs(x0, C.byref(c.params))
        finally:
            O.orc().orc_set_profile(0, 0, 0, 0, 0, 0)
        got = list(out)
        want = [ref.sigma_u2, ref.lambda_, ref.sigma, ref.dsigma_u2]
        assert np.array(got).tobytes() == np.array(want).tobytes(), (trial, prof, x0, got, want)
        cases += 1
    assert cases == 400


@pytest.mark.parametrize("x_adapt", [-0.05, -0.0, 0.0, 1.5])
def test_adaptive_reference_height_validated(x_adapt):
    """SampleOptions::x_adapt outside (0, H] is rejected when the problem is
    built (the fast path may therefore assume x_adapt in the layer)."""
    opt = ablmc.SampleOptions(adaptive=True, x_adapt=x_adapt)
    with pytest.raises(ValueError, match="x_adapt"):
        ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.gl, ablmc.QoISpec(), 0.3, 0.1,
                           1.0, 8, 3, opt)


@pytest.mark.parametrize("field,value", [("l_max", capi.ABLMC_MAX_LEVELS), ("l_max", -1),
                                         ("pilot_levels_max", capi.ABLMC_MAX_LEVELS)])
def test_run_mlmc_refuses_levels_beyond_the_result_rows(field, value):
    """ablmc_run_result has ABLMC_MAX_LEVELS per-level rows: options that could
    produce more are an invalid argument (no truncation), checked before the
    device is touched."""
    pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.gl, ablmc.QoISpec(), 0.5, 0.1,
                            1.0, 1, 1)
    o = ablmc.MlmcOptions(**{field: value})
    with pytest.raises(ValueError, match="l_max and pilot_levels_max"):
        ablmc.run_mlmc(pr, 1e-3, o)

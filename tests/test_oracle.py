"""Pins the C restatement (oracle/ablmc_oracle.c) before it is trusted.

1. Against the reference's own golden values (tests/golden/reference_goldens.json,
   copied from /root/reference/proj/tests with file:line and tolerance).
2. Bit-for-bit against outputs of the unmodified reference
   (tests/golden/ref_vectors.json, made by tests/golden/make_ref_vectors.py).
3. Live against oracle/_ref/libablmc_ref.so on fresh random inputs, when built.
CPU only.
"""
import ctypes as C
import math

import numpy as np
import pytest

import oracle_lib as O
from conftest import fx
from paper_1612_07717_b200 import capi

P = C.POINTER
IG = {"se": 0, "gl": 1, "baoab": 2}


def rel_close(a, b, rel):
    return abs(a - b) <= rel * abs(b)


# ---------------------------------------------------------------- goldens
def test_philox_known_answers(goldens):
    for ctr, key, want in goldens["philox_kat"]["cases"]:
        o = (C.c_uint32 * 4)()
        O.orc().orc_philox4x32((C.c_uint32 * 4)(*ctr), (C.c_uint32 * 2)(*key), o)
        assert list(o) == want


def test_stream_known_answers(goldens):
    k = goldens["stream_kat"]
    key = (C.c_uint32 * 2)()
    O.orc().orc_stream_key(k["seed"], k["level"], key)
    assert [f"{key[0]:08x}", f"{key[1]:08x}"] == k["key_hex"]
    z = O.orc_normals(k["seed"], k["level"], k["idx"], 0, 3)
    assert list(z) == k["normals"]


def test_profile_goldens(goldens):
    g = goldens["profiles"]
    p = O.default_params()
    co = lambda x: O.orc().orc_sde_coeffs(x, C.byref(p))  # noqa: E731
    for x, want in g["sigma_u"]:
        assert rel_close(math.sqrt(co(x).sigma_u2), want, 1e-12)
    for x, want in g["tau"]:
        assert rel_close(1.0 / co(x).lambda_, want, 1e-12)
    for x, want in g["lambda"]:
        assert rel_close(co(x).lambda_, want, 1e-12)
    for x, want in g["diffusion_sigma"]:
        assert rel_close(co(x).sigma, want, 1e-12)


def test_drift_goldens(goldens):
    g = goldens["dV_dX"]
    p = O.default_params()
    for x, u, want in g["values"]:
        c = O.orc().orc_sde_coeffs(x, C.byref(p))
        assert rel_close(O.orc().orc_dv_dx(C.byref(c), u), want, 1e-12)
    for x, u in g["zeros"]:
        c = O.orc().orc_sde_coeffs(x, C.byref(p))
        assert O.orc().orc_dv_dx(C.byref(c), u) == 0.0


def test_one_step_goldens(goldens):
    g = goldens["one_step"]
    p = O.default_params()
    for ig, xi, wx, wu in g["cases"]:
        s = O.OrcState(g["x0"], g["u0"], 1, 0)
        pan = C.c_int()
        assert O.orc().orc_step(IG[ig], C.byref(s), g["h"], xi, C.byref(p), 0, C.byref(pan)) == 0
        assert rel_close(s.x, wx, 1e-12) and rel_close(s.u, wu, 1e-12), ig


def test_se_stability_limit(goldens):
    p = O.default_params()
    assert rel_close(O.orc().orc_se_stability_limit(C.byref(p)),
                     goldens["se_stability_limit"]["value"], 1e-12)


def test_reflection_cases(goldens):
    for (x, u, H, par, nr), (wx, wu, wcount, wpar, wnr) in goldens["reflection"]["cases"]:
        xx, uu, pp, nn, cc = C.c_double(x), C.c_double(u), C.c_int(par), C.c_int64(nr), C.c_int()
        assert O.orc().orc_reflect(C.byref(xx), C.byref(uu), H, C.byref(pp), C.byref(nn),
                                   C.byref(cc)) == 0
        assert rel_close(xx.value, wx, 1e-14)
        assert (uu.value, cc.value, pp.value, nn.value) == (wu, wcount, wpar, wnr)
    for x, u, H, par, nr in goldens["reflection"]["unstable"]:
        xx, uu = C.c_double(float(x)), C.c_double(u)
        pp, nn = C.c_int(par), C.c_int64(nr)
        assert O.orc().orc_reflect(C.byref(xx), C.byref(uu), H, C.byref(pp), C.byref(nn), None) == -1


def test_coarse_noise_goldens(goldens):
    g = goldens["coarse_noise"]
    for a, b, s0, s1, sc, want in g["se"]:
        v = O.orc().orc_coarse_noise_se(a, b, s0, s1, sc)
        assert v == want if want == 0.0 else rel_close(v, want, 1e-12)
    for a, b, lam, h, s0, s1, sc, want in g["gl"]:
        assert rel_close(O.orc().orc_coarse_noise_gl(a, b, lam, h, s0, s1, sc), want, 1e-12)
    # lambda h -> 0 reduces to the Brownian-bridge rule (test_noise.cpp:412-413)
    assert rel_close(O.orc().orc_coarse_noise_gl(0.3, -0.5, 1e-14, 0.0125, 1, -1, -1),
                     O.orc().orc_coarse_noise_se(0.3, -0.5, 1, -1, -1), 1e-10)


def test_smoothing_polynomial_goldens(goldens):
    g = goldens["smoothing_polynomial"]
    for r in (0, 1, 2, 4):
        c = (C.c_double * (r + 2))()
        assert O.orc().orc_build_smoothing_polynomial(r, c) == 0
        for got, want in zip(c, g[f"r{r}"]):
            if want is not None:
                assert abs(got - want) <= 1e-12
    assert O.orc().orc_build_smoothing_polynomial(13, (C.c_double * 16)()) != 0
    assert O.orc().orc_build_smoothing_polynomial(-1, (C.c_double * 16)()) != 0


def test_constant_qoi_difference_is_zero(goldens):
    g = goldens["coupled_constant_qoi"]
    edges = (C.c_double * 2)(0.0, 1.0)
    for ig in (0, 1, 2):
        pr = capi.ProblemC()
        pr.params = O.default_params()
        pr.integrator, pr.signs_on = ig, 1
        pr.qoi.kind, pr.qoi.r, pr.qoi.delta, pr.qoi.n_edges = 3, 4, 0.1, 2
        pr.qoi.bin_edges = C.cast(edges, P(C.c_double))
        pr.x0, pr.u0, pr.T, pr.m0, pr.seed = 0.05, 0.1, 1.0, g["m0"], g["seed"]
        st = O.Stats(1)
        assert O.orc().orc_accumulate_samples(C.byref(pr), g["level"], g["idx"], 1, C.byref(st.c)) == 0
        assert st.n == 1 and st.cost_steps == g["steps"] and st.sum_y[0] == 0.0


# ------------------------------------------------ bit-exact vs the reference
def test_normals_bit_exact(ref_vectors):
    for s in ref_vectors["normals"]:
        z = O.orc_normals(s["seed"], s["level"], s["idx"], s["k0"], len(s["z"]))
        assert [v.hex() for v in z] == s["z"]


@pytest.mark.parametrize("idx,k0", [(2**32 - 1, 0), (2**32, 6), (2**40 + 3, 1), (2**63 + 5, 2),
                                    (12345, 2**33 - 2), (7, 2**33 + 1)])
def test_normals_bit_exact_high_counter_words(idx, k0):
    """Sample indices and draw numbers whose Philox counter words above 32
    bits are nonzero (noise.hpp:63-70: ctr = (k>>1, k>>33, idx, idx>>32)),
    live against the reference itself (oracle/_ref)."""
    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    z = O.orc_normals(42, 3, idx, k0, 6)
    r = O.ref_normals(42, 3, idx, k0, 6)
    assert [v.hex() for v in z] == [v.hex() for v in r]


def test_sde_coeffs_bit_exact(ref_vectors):
    p = O.default_params()
    for e in ref_vectors["sde_coeffs"]:
        c = O.orc().orc_sde_coeffs(fx(e["x"]), C.byref(p))
        assert [c.sigma_u2, c.lambda_, c.sigma, c.dsigma_u2] == [fx(v) for v in e["c"]]


def test_steps_bit_exact(ref_vectors):
    p = O.default_params()
    for e in ref_vectors["steps"]:
        x, u, par, nr = e["in"]
        s = O.OrcState(fx(x), fx(u), par, nr)
        pan = C.c_int()
        rc = O.orc().orc_step(e["ig"], C.byref(s), fx(e["h"]), fx(e["xi"]), C.byref(p), e["scale"],
                              C.byref(pan))
        assert rc == e["rc"]
        if rc == 0:
            ox, ou, opar, onr, opan = e["out"]
            assert (s.x, s.u, s.parity, s.n_refl, pan.value) == (fx(ox), fx(ou), opar, onr, opan)


def _params(d):
    return O.default_params(**{k: d[k] for k in ("kappa_sigma", "kappa_tau", "u_star", "H",
                                                   "eps_reg", "x_ref", "noise_scale")})


def test_pairs_bit_exact(ref_vectors):
    for case in ref_vectors["pairs"]:
        d = case["problem"]
        p = _params(d)
        M = d["m0"] << case["level"]
        for i, st in enumerate(case["states"]):
            if d.get("adaptive"):
                rc, f, c, _ = O.orc_pair_adaptive(d["integrator"], p, d["x0"], d["u0"], d["T"],
                                                  d["T"] / M, d["x_adapt"], d["seed"],
                                                  case["level"], case["first"] + i,
                                                  signs_on=d["signs_on"])
            else:
                rc, f, c = O.orc_pair(d["integrator"], p, d["x0"], d["u0"], d["T"], M, d["seed"],
                                      case["level"], case["first"] + i, signs_on=d["signs_on"])
            assert (rc == 0) == bool(st[4]), case["name"]
            if rc == 0:
                got = [f.x.hex(), f.u.hex(), f.parity, f.n_refl, 1, c.x.hex(), c.u.hex(), c.parity,
                       c.n_refl, 1]
                assert got == st, (case["name"], i)


def test_paths_bit_exact(ref_vectors):
    for case in ref_vectors["paths"]:
        d = case["problem"]
        p = _params(d)
        for i, st in enumerate(case["states"]):
            if d.get("adaptive"):
                rc, s, _ = O.orc_path_adaptive(d["integrator"], p, d["x0"], d["u0"], d["T"],
                                               d["T"] / case["M"], d["x_adapt"], d["seed"],
                                               case["stream_level"], case["first"] + i)
            else:
                rc, s = O.orc_path(d["integrator"], p, d["x0"], d["u0"], d["T"], case["M"],
                                   d["seed"], case["stream_level"], case["first"] + i)
            assert rc == 0 and [s.x.hex(), s.u.hex(), s.parity, s.n_refl, 1] == st


def problem_from(d):
    pr = capi.ProblemC()
    pr.params = _params(d)
    pr.integrator, pr.signs_on = d["integrator"], d["signs_on"]
    pr.qoi.kind, pr.qoi.a, pr.qoi.b, pr.qoi.r, pr.qoi.delta = d["qoi_kind"], 0.1055, 0.1555, 4, 0.1
    keep = None
    if d["qoi_kind"] == 3:
        keep = (C.c_double * len(d["edges"]))(*d["edges"])
        pr.qoi.n_edges = len(d["edges"])
        pr.qoi.bin_edges = C.cast(keep, P(C.c_double))
    pr.x0, pr.u0, pr.T, pr.m0, pr.seed = d["x0"], d["u0"], d["T"], d["m0"], d["seed"]
    pr.adaptive, pr.x_adapt = d.get("adaptive", 0), d.get("x_adapt", 0.05)
    return pr, keep


def test_accumulate_bit_exact(ref_vectors):
    for case in ref_vectors["accumulate"]:
        pr, keep = problem_from(case["problem"])
        dim = len(case["sum_y"])
        st = O.Stats(dim)
        assert O.orc().orc_accumulate_samples(C.byref(pr), case["level"], case["first"],
                                              case["count"], C.byref(st.c)) == 0
        assert [v.hex() for v in st.sum_y] == case["sum_y"]
        assert [v.hex() for v in st.sum_y2] == case["sum_y2"]
        assert (st.n, st.failed, st.cost_steps) == (case["n"], case["failed"], case["cost_steps"])


# ---------------------------------------------------- live vs the reference
needs_ref = pytest.mark.skipif(O.ref() is None, reason="oracle/_ref not built")


@needs_ref
def test_live_pairs_random_configs():
    rng = np.random.default_rng(11)
    R = O.ref()
    for trial in range(12):
        ig = trial % 3
        pr = capi.ProblemC()
        pr.params = O.default_params(u_star=float(rng.choice([0.2, 0.6, 1.0])),
                                     eps_reg=float(rng.choice([0.01, 0.05])))
        pr.integrator, pr.signs_on = ig, int(rng.integers(0, 2))
        pr.x0, pr.u0 = float(rng.uniform(0.01, 0.99)), float(rng.normal(0, 0.3))
        pr.T, pr.m0 = 1.0, int(rng.choice([4, 16, 40]))
        pr.seed = int(rng.integers(0, 2**63))
        level = int(rng.integers(1, 5))
        arr = (capi.PairStateC * 16)()
        R.ref_pair_states(C.byref(pr), level, 100, 16, arr)
        M = pr.m0 << level
        for i in range(16):
            rc, f, c = O.orc_pair(ig, pr.params, pr.x0, pr.u0, pr.T, M, pr.seed, level, 100 + i,
                                  signs_on=pr.signs_on)
            assert (rc == 0) == bool(arr[i].fine.ok)
            if rc == 0:
                assert (f.x, f.u, f.parity, f.n_refl) == (arr[i].fine.x, arr[i].fine.u,
                                                          arr[i].fine.parity, arr[i].fine.n_refl)
                assert (c.x, c.u, c.parity, c.n_refl) == (arr[i].coarse.x, arr[i].coarse.u,
                                                          arr[i].coarse.parity, arr[i].coarse.n_refl)


@needs_ref
def test_live_explicit_xi_matches_reference_steps():
    """Oracle mode (host-supplied xi) == a path driven step by step through the
    reference's own step() with the same xi, including heavy reflection."""
    rng = np.random.default_rng(5)
    R = O.ref()
    p = O.default_params(u_star=1.0)
    for ig in (0, 1, 2):
        for _ in range(5):
            M = 200
            xi = rng.normal(size=M) * 1.5
            rc, s = O.orc_path(ig, p, 0.5, 0.0, 1.0, M, 0, 0, 0, xi=xi)
            st = capi.PathStateC(0.5, 0.0, 1, 1, 0)
            ok = 0
            for k in range(M):
                ok = R.ref_step(ig, C.byref(st), 1.0 / M, float(xi[k]), C.byref(p), 0, None)
                if ok != 0:
                    break
            assert (rc == 0) == (ok == 0)
            if rc == 0:
                assert (s.x, s.u, s.parity, s.n_refl) == (st.x, st.u, st.parity, st.n_refl)


@needs_ref
def test_live_accumulate_vs_reference_multiworker():
    """orc accumulate == reference accumulate_samples with 3 worker threads."""
    R = O.ref()
    for ig in (0, 1, 2):
        pr = capi.ProblemC()
        pr.params = O.default_params()
        pr.integrator, pr.signs_on = ig, 1
        pr.qoi.kind, pr.qoi.r, pr.qoi.delta = 0, 4, 0.1
        pr.x0, pr.u0, pr.T, pr.m0, pr.seed = 0.05, 0.1, 1.0, 20, 77
        a, b = O.Stats(1), O.Stats(1)
        assert O.orc().orc_accumulate_samples(C.byref(pr), 1, 0, 20000, C.byref(a.c)) == 0
        assert R.ref_accumulate_samples(C.byref(pr), 1, 0, 20000, 3, C.byref(b.c), None) == 0
        assert a.sum_y[0] == b.sum_y[0] and a.sum_y2[0] == b.sum_y2[0]
        assert (a.n, a.cost_steps) == (b.n, b.cost_steps)

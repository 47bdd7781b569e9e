"""The reference's noise and one-step statistical tests on the device's Philox /
Box-Muller and steps (tests/test_noise.cpp:30-101, test_integrators.cpp:121-149):
stream determinism, empirical moments, independence across sample indices,
KS normality with sign flips, and the exact OU one-step law of the O-step."""
import math

import numpy as np
import pytest
from scipy import stats

import oracle_lib as O
from paper_1612_07717_b200 import ablmc

pytestmark = pytest.mark.gpu
Ig = ablmc.Integrator


def test_streams_are_deterministic_functions_of_their_identifiers():
    """test_noise.cpp:30-51."""
    a = ablmc.normals(42, 3, 17, 0, 1000)
    assert np.array_equal(a, ablmc.normals(42, 3, 17, 0, 1000))
    # indexed access agrees with sequential draws, any offset and order
    for k0 in (63, 17, 0, 999):
        assert ablmc.normals(42, 3, 17, k0, 1)[0] == a[k0]
    base = a[:16]
    assert not np.array_equal(base, ablmc.normals(42, 3, 18, 0, 16))
    assert not np.array_equal(base, ablmc.normals(42, 4, 17, 0, 16))
    assert not np.array_equal(base, ablmc.normals(43, 3, 17, 0, 16))
    # and they are the reference's stream to within ulps (Box-Muller math)
    assert np.allclose(base, O.orc_normals(42, 3, 17, 0, 16), rtol=1e-13, atol=1e-15)


def test_empirical_moments_over_1e6_draws():
    """test_noise.cpp:53-66."""
    z = ablmc.normals(12345, 0, 0, 0, 1000000)
    assert abs(z.mean()) <= 4e-3
    assert abs(z.var(ddof=1) - 1.0) <= 6e-3


def test_streams_with_different_sample_indices_are_uncorrelated():
    """test_noise.cpp:68-86 (draw 0 of streams (777, 2, i) and (777, 2, i+1))."""
    n = 100000
    x = np.array([ablmc.normals(777, 2, i, 0, 2)[0] for i in range(n + 1)])
    rho = np.corrcoef(x[:-1], x[1:])[0, 1]
    assert abs(rho) < 0.01


def test_sign_flips_preserve_the_standard_normal_law():
    """test_noise.cpp:88-101."""
    z = ablmc.normals(31415, 1, 9, 0, 100000)
    flipped = np.where(np.arange(z.size) % 2 == 0, -z, z)
    assert stats.kstest(z, "norm").pvalue > 0.01
    assert stats.kstest(flipped, "norm").pvalue > 0.01


@pytest.mark.parametrize("ig", [Ig.gl, Ig.baoab])
def test_o_step_reproduces_the_exact_ou_one_step_law(ig):
    """test_integrators.cpp:121-149: eps_reg = 0.45 freezes the coefficients
    over everything the step reaches, so one GL / BAOAB step of h = 0.02 from
    (0.2, 0.3) is the exact OU kernel in U: mean and variance over 1e6
    paths within 4 standard errors."""
    mp = ablmc.ModelParams(eps_reg=0.45)
    x, u0, h = 0.2, 0.3, 0.02
    c = O.orc().orc_sde_coeffs(x, O.default_params(eps_reg=0.45))
    lam = getattr(c, O.OrcCoeffs._fields_[1][0])
    sig = getattr(c, O.OrcCoeffs._fields_[2][0])
    exact_mean = math.exp(-lam * h) * u0
    exact_sd = sig * math.sqrt(-math.expm1(-2.0 * lam * h) / (2.0 * lam))
    pr = ablmc.Problem.make(mp, ig, ablmc.QoISpec(), x, u0, h, 1, 7)
    n = 1000000
    got = ablmc.simulate_paths(pr, 1, 0, n, 1 if ig == Ig.gl else 2)
    assert got["ok"].all()
    u = got["u"]
    assert abs(u.mean() - exact_mean) <= 4.0 * exact_sd / math.sqrt(n)
    assert abs(u.var(ddof=1) - exact_sd ** 2) <= 4.0 * exact_sd ** 2 * math.sqrt(2.0 / (n - 1))
